"""the reference's two callers, switched to the B200 backend.

Both callers of the hot path -- the batch CLI `bisimp.cli._execute`
(cli.py:52-84) and the service worker `Session._run_worker`
(service/sessions.py:87-115) -- are run from the UNMODIFIED reference in
`baseline/_ref`, with the one-line switch INTEGRATION.md §1 documents: the
name `run` they imported from `bisimp.solvers` is bound to this package's
`run` instead.  Their artefacts are compared with the stock reference's:

* CLI: problem.json byte-identical, every PGM (snapshots and final)
  byte-identical, convergence.csv / summary.json equal to the float
  tolerance of the trajectory contract, and byte-deterministic across two
  B200 runs (the reference's tests/test_cli.py:85-90 property).
* Service: the same frames published (iterations, float32 payload bytes,
  scalars), final status, and clock=time.perf_counter (the worker's clock,
  sessions.py:107) served from device stamps without per-iteration syncs.
"""
import json
import os
import sys
import time
import warnings

import numpy as np
import pytest

from conftest import ROOT

REF_DIR = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.gpu
warnings.filterwarnings("ignore", message="decay exponent")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF_DIR, "bisimp")):
        pytest.skip("baseline/_ref (the vendored reference) is not installed")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import bisimp.cli
    import bisimp.service.sessions
    return bisimp


@pytest.fixture(scope="module")
def B():
    import paper_2204_06204_b200 as B
    return B


CLI_ARGS = ["bench", "run", "teaser", "--algo", "pfbto", "--scale", "0.25", "--max-iters", "300",
            "--snapshot-every", "100"]


def _cli(ref, out, monkeypatch=None, backend=None):
    if backend is not None:
        monkeypatch.setattr(ref.cli, "run", backend)   # the INTEGRATION.md §1 switch
    try:
        rc = ref.cli.main(CLI_ARGS + ["--out", str(out)])
    finally:
        if backend is not None:
            monkeypatch.undo()
    return rc, {p: (out / p).read_bytes() for p in sorted(os.listdir(out))}


def _csv(b):
    lines = b.decode().strip().split("\n")
    return lines[0], np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])


def test_cli_execute_with_b200_backend(ref, B, tmp_path, monkeypatch, capsys):
    rc_ref, want = _cli(ref, tmp_path / "ref")
    rc1, got = _cli(ref, tmp_path / "b200_1", monkeypatch, B.run)
    rc2, again = _cli(ref, tmp_path / "b200_2", monkeypatch, B.run)
    capsys.readouterr()
    assert rc_ref == rc1 == rc2 == 2  # budget
    assert sorted(got) == sorted(want) == sorted(again)
    assert sorted(got) == ["convergence.csv", "density_000100.pgm", "density_000200.pgm",
                           "density_000300.pgm", "final_density.pgm", "problem.json",
                           "summary.json"]
    # byte-deterministic through the B200 backend (test_cli.py:85-90)
    assert got == again
    # identical images and problem document
    for name in got:
        if name.endswith(".pgm") or name == "problem.json":
            assert got[name] == want[name], name
    h1, c1 = _csv(got["convergence.csv"])
    h0, c0 = _csv(want["convergence.csv"])
    assert h1 == h0 and c1.shape == c0.shape
    assert np.array_equal(c1[:, 0], c0[:, 0]) and np.all(c1[:, 1] == 0.0)  # clock=None -> 0.0
    np.testing.assert_allclose(c1[:, 2:], c0[:, 2:], rtol=1e-9, atol=1e-14)
    s1, s0 = json.loads(got["summary.json"]), json.loads(want["summary.json"])
    assert s1.keys() == s0.keys() and s1["config"] == s0["config"]
    assert s1["reason"] == s0["reason"] and s1["iterations"] == s0["iterations"]
    for key in ("compliance", "volume", "residual_inf"):
        assert s1[key] == pytest.approx(s0[key], rel=1e-9)


def _session_run(ref, problem, config, backend=None, monkeypatch=None):
    sessions = ref.service.sessions
    if backend is not None:
        monkeypatch.setattr(sessions, "run", backend)   # the INTEGRATION.md §1 switch
    try:
        s = sessions.Session(config=config)
        frames = []
        publish = s.slot.publish
        s.slot.publish = lambda f: (frames.append(f), publish(f))
        s.set_problem(problem)
        t0 = time.perf_counter()
        s.start()
        s._worker.join(timeout=300)
        wall = time.perf_counter() - t0
        assert not s._worker.is_alive()
    finally:
        if backend is not None:
            monkeypatch.undo()
    return s, frames, wall


def test_session_worker_with_b200_backend(ref, B, monkeypatch):
    problem = ref.problems.catalog()["lshape"].scale(0.25)
    config = ref.solvers.SolverConfig(algorithm="pfbto_jacobi", max_iters=400, snapshot_every=50)
    s_ref, f_ref, _ = _session_run(ref, problem, config)
    s_b, f_b, _ = _session_run(ref, problem, config, B.run, monkeypatch)
    assert s_b.status == s_ref.status == "budget"
    assert s_b.error_message is None
    assert [f.iter for f in f_b] == [f.iter for f in f_ref] == list(range(50, 401, 50))
    for fb, fr in zip(f_b, f_ref):
        assert (fb.nx, fb.ny) == (fr.nx, fr.ny)
        assert fb.payload == fr.payload, fb.iter        # float32 bytes of v_phys
        assert fb.compliance == pytest.approx(fr.compliance, rel=1e-9)
        assert fb.volume == pytest.approx(fr.volume, rel=1e-12)
    st = s_b.state_view()
    assert st["iter"] == 400 and st["status"] == "budget"


def test_realtime_clock_is_stamped_on_device(B):
    """clock=time.perf_counter (the service's clock) keeps the batched device
    loop: elapsed_s comes from per-iteration device stamps mapped onto the
    clock, monotone, inside the run's wall-time window."""
    spec = B.problems.mbb_half_beam(440, 250)
    cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=3000)
    B.run(spec, B.SolverConfig(algorithm="pfbto_jacobi", max_iters=50))  # warm
    t_a = time.perf_counter()
    res = B.run(spec, cfg, clock=time.perf_counter)
    t_b = time.perf_counter()
    el = np.asarray(res.record.elapsed_s)
    assert len(el) == 3000
    assert np.all(np.diff(el) >= 0.0) and el[0] > 0.0
    assert el[-1] <= t_b - t_a
    per_iter = np.median(np.diff(el))
    assert 0.0 < per_iter < 2e-4, per_iter          # device time per C2 iteration, not a sync
    # the same run without a clock: identical numbers
    plain = B.run(spec, cfg)
    assert plain.record.compliance == res.record.compliance
    # a custom (non real-time) clock is called once per completed iteration
    calls = []
    res2 = B.run(spec, B.SolverConfig(algorithm="pfbto_jacobi", max_iters=20),
                 clock=lambda: calls.append(1) or float(len(calls)))
    assert len(calls) == 21 and res2.record.elapsed_s == [float(i) for i in range(1, 21)]
