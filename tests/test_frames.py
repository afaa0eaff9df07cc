"""Density frames converted on the device: the service's
float32 payload (service/sessions.py:97) and the CLI's PGM snapshot
(outputs.py:21-30), byte-identical to the reference's host conversions.

GPU tests compare against the golden bytes written by the real reference
(tests/golden/make_golden.py::make_frames) and against the oracle
restatement (oracle/bisimp_oracle.py pgm_bytes / frame_payload)."""
import os

import numpy as np
import pytest

from oracle import bisimp_oracle as O

from conftest import GOLDEN


@pytest.fixture(scope="module")
def B():
    import paper_2204_06204_b200 as B
    return B


@pytest.fixture(scope="module")
def Z():
    return np.load(os.path.join(GOLDEN, "frames.npz"), allow_pickle=False)


def small_problem(B, nx=8, ny=8, volume_fraction=0.4):
    return B.ProblemSpec(nx=nx, ny=ny, volume_fraction=volume_fraction,
                         fixtures=({"edge": "left", "dofs": "xy"},),
                         loads=({"point": (1.0, 0.5), "fy": -1.0},))


def test_frame_kinds_validated_on_cpu():
    # host-side validation only: no device call happens before the kind check
    from paper_2204_06204_b200 import outputs, solvers
    assert outputs.FRAME_KINDS == {"f32": 0, "pgm": 1}
    with pytest.raises(ValueError, match="unknown frame kind"):
        solvers.run(None, solvers.SolverConfig(), frame_kind="png")
    f = outputs.Frame(iter=1, compliance=1.0, residual_inf=0.0, volume=1.0, nx=1, ny=1,
                      payload=b"\0", kind="f32")
    with pytest.raises(ValueError, match="expected 'pgm'"):
        outputs.write_frame_pgm(f, "/nonexistent/x.pgm")


@pytest.mark.gpu
def test_payload_matches_reference_bytes(B, Z):
    from paper_2204_06204_b200.outputs import frame_payload
    assert frame_payload(Z["f32_values"]) == Z["f32_payload"].tobytes()
    assert frame_payload(Z["design_v_phys"]) == Z["design_payload"].tobytes()
    import torch
    t = torch.from_numpy(Z["design_v_phys"]).cuda()
    assert frame_payload(t) == Z["design_payload"].tobytes()
    # every length mod 4 and an unaligned tail
    for n in (0, 1, 2, 3, 5, 7, 1027):
        v = Z["f32_values"][:n]
        assert frame_payload(v) == O.frame_payload(v)


@pytest.mark.gpu
def test_pixels_match_reference_bytes(B, Z, tmp_path):
    from paper_2204_06204_b200 import outputs
    for name, v in (("design", Z["design_v_phys"]), ("px", Z["px_values"])):
        nx, ny = int(Z[f"{name}_nx"]), int(Z[f"{name}_ny"])
        path = tmp_path / f"{name}.pgm"
        outputs.write_snapshot(v, nx, ny, path)
        assert path.read_bytes() == Z[f"{name}_pgm"].tobytes()
        assert path.read_bytes() == O.pgm_bytes(v, nx, ny)
    import torch
    px = outputs.density_pixels(torch.from_numpy(Z["px_values"]).cuda())
    assert px.is_cuda and px.dtype == torch.uint8
    hdr = len(outputs.pgm_header(int(Z["px_nx"]), 1))
    assert px.cpu().numpy().tobytes() == Z["px_pgm"].tobytes()[hdr:]


@pytest.mark.gpu
def test_snapshot_validation(B, tmp_path):
    from paper_2204_06204_b200 import outputs
    with pytest.raises(ValueError, match="field has length"):
        outputs.write_snapshot(np.full(5, 0.5), 2, 2, tmp_path / "a.pgm")
    for bad in (np.array([0.5, 1.0 + 1e-16 * 3, 0.2]), np.array([0.5, -1e-300, 0.2])):
        with pytest.raises(ValueError, match=r"must lie in \[0, 1\]"):
            outputs.write_snapshot(bad, 3, 1, tmp_path / "b.pgm")
        assert not (tmp_path / "b.pgm").exists()
        with pytest.raises(ValueError):
            O.pgm_bytes(bad, 3, 1)
    with pytest.raises(ValueError):
        outputs.write_snapshot(np.zeros(0), 0, 3, tmp_path / "c.pgm")


@pytest.mark.gpu
@pytest.mark.parametrize("algorithm", ["pfbto_jacobi", "cpfbto_krylov", "pgd_exact"])
def test_run_frame_sink_cadence_and_bytes(B, algorithm):
    """frame_sink sees exactly the sink's iterations, and its payload is the
    sink state's v_phys converted as the service / CLI would."""
    cfg = B.SolverConfig(algorithm=algorithm, max_iters=25, snapshot_every=10)
    prob = small_problem(B, 12, 8)
    for kind in ("f32", "pgm"):
        states, frames = [], []
        res = B.run(prob, cfg, sink=states.append, frame_sink=frames.append, frame_kind=kind)
        assert [s.iter for s in states] == [10, 20, 25] == [f.iter for f in frames]
        for s, f in zip(states, frames):
            assert f.kind == kind and (f.nx, f.ny) == (12, 8)
            assert f.compliance == s.compliance and f.residual_inf == s.residual_inf
            assert f.volume == pytest.approx(s.volume, rel=1e-14)
            if kind == "f32":
                assert f.payload == O.frame_payload(s.v_phys)
            else:
                assert f.payload == O.pgm_bytes(s.v_phys, 12, 8)[len(b"P5\n12 8\n255\n"):]
        assert res.state.iter == 25
        # frames alone (no state sink), same bytes
        only = []
        B.run(prob, cfg, frame_sink=only.append, frame_kind=kind)
        assert [f.payload for f in only] == [f.payload for f in frames]


@pytest.mark.gpu
def test_run_frame_sink_zero_iterations(B):
    frames = []
    res = B.run(small_problem(B, 4, 4), B.SolverConfig(max_iters=0), frame_sink=frames.append)
    assert [f.iter for f in frames] == [0]
    assert frames[0].payload == O.frame_payload(res.state.v_phys)


@pytest.mark.gpu
def test_write_frame_pgm_equals_write_snapshot(B, tmp_path):
    from paper_2204_06204_b200 import outputs
    frames = []
    res = B.run(small_problem(B, 10, 6), B.SolverConfig(max_iters=7),
                frame_sink=frames.append, frame_kind="pgm")
    outputs.write_frame_pgm(frames[-1], tmp_path / "f.pgm")
    outputs.write_snapshot(res.state.v_phys, 10, 6, tmp_path / "s.pgm")
    assert (tmp_path / "f.pgm").read_bytes() == (tmp_path / "s.pgm").read_bytes()


@pytest.mark.gpu
def test_read_frame_needs_a_completed_iteration(B):
    from paper_2204_06204_b200 import solvers as S
    spec = small_problem(B, 6, 4)
    cfg = B.SolverConfig(max_iters=10)
    loop = S.DeviceLoop(S._prepare(spec, cfg), cfg, max_batch=4)
    with pytest.raises(ValueError, match="no completed iteration"):
        loop.read_frame("f32")
    done, status, _ = loop.run(1, [cfg.step_size(k) for k in range(1, 4)])
    assert done == 3
    _, _, vp, _ = loop.read_state()
    assert loop.read_frame("f32") == O.frame_payload(vp)
    assert loop.read_frame("pgm") == O.pgm_bytes(vp, 6, 4)[len(b"P5\n6 4\n255\n"):]
