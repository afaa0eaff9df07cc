"""The drop-in boundary with the reference's OWN objects.

The reference's callers build `bisimp.problems.ProblemSpec`,
`bisimp.solvers.SolverConfig` (cli.py:55-62, service/sessions.py:106-107) and
`bisimp.fea.GridModel` (via `problems.resolve`), then call the solver API.
These tests pass exactly those objects -- imported from the unmodified
reference installed in `baseline/_ref` (git-ignored, shipped to the GPU box)
-- to this package and compare with the reference's own answers.  The
INTEGRATION.md §2 ctypes snippet is executed verbatim.

`baseline/_ref` is produced by
    python -m pip install --no-index --no-build-isolation --no-deps \\
        --target baseline/_ref <copy of /root/reference/pkg>
(DESIGN.md §9).  Without it the tests skip (they never read /root/reference).
"""
import os
import re
import sys
import warnings

import numpy as np
import pytest

from conftest import ROOT

REF_DIR = os.path.join(ROOT, "baseline", "_ref")

warnings.filterwarnings("ignore", message="decay exponent")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF_DIR, "bisimp")):
        pytest.skip("baseline/_ref (the vendored reference) is not installed")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import bisimp.fea
    import bisimp.filtering
    import bisimp.problems
    import bisimp.projection
    import bisimp.solvers
    return bisimp


@pytest.fixture(scope="module")
def B():
    import paper_2204_06204_b200 as B
    return B


def mbb(ref_problems, nx=48, ny=24):
    return ref_problems.ProblemSpec(
        nx=nx, ny=ny, volume_fraction=0.5,
        fixtures=({"edge": "left", "dofs": "x"}, {"point": (1.0, 1.0), "dofs": "y"}),
        loads=({"edge": "top", "span": (0.0, 0.02), "fy": -1.0},))


# ------------------------------------------------------------------- CPU ---

def test_reference_config_normalised(ref, B):
    """A reference SolverConfig (reference fields only) becomes this package's
    config with the approximate-inverse knobs at their defaults."""
    from paper_2204_06204_b200.solvers import as_solver_config
    rc = ref.solvers.SolverConfig(algorithm="pfbto_jacobi", alpha0=0.2, max_iters=7, m=0.8,
                                  snapshot_every=3, seed=5, mean_projection=False)
    assert not hasattr(rc, "inner_steps")
    c = as_solver_config(rc)
    assert isinstance(c, B.SolverConfig)
    for name in ("algorithm", "alpha0", "m", "beta", "krylov_dim", "eta", "max_iters", "tol_dv",
                 "tol_res", "snapshot_every", "seed", "mean_projection"):
        assert getattr(c, name) == getattr(rc, name), name
    assert c.resolved_inner_steps() == 0 and c.mg_omega == 0.6 and c.mg_smooth is None
    assert c.step_size(9) == rc.step_size(9)
    with pytest.raises(TypeError):
        as_solver_config(object())


def test_integration_snippet_struct_matches_header():
    """INTEGRATION.md §2's ctypes Cfg is a prefix of bsp_solver_config with
    struct_size first, and _native's full struct matches the header order."""
    from paper_2204_06204_b200._native import SolverConfigC
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    snippet = re.search(r"```python\nimport ctypes as C, numpy as np\n(.*?)```", text, re.S).group(1)
    fields = re.findall(r'\("(\w+)",', snippet.split("class Cfg")[1].split("spec =")[0])
    full = [f[0] for f in SolverConfigC._fields_]
    assert fields[0] == "struct_size" and fields == full[:len(fields)]
    hdr = open(os.path.join(ROOT, "include", "bisimp_b200.h")).read()
    body = hdr[hdr.index("typedef struct bsp_solver_config {"):hdr.index("} bsp_solver_config;")]
    names = [n for part in re.findall(r"^\s+(?:const )?\w+\*? +([\w, *]+);", body, re.M)
             for n in re.split(r",\s*", part.replace("*", ""))]
    assert names == full


# ------------------------------------------------------------------- GPU ---

@pytest.mark.gpu
def test_run_with_reference_problem_and_config(ref, B):
    """run(ref ProblemSpec, ref SolverConfig) == the reference's run, 60 iterations."""
    spec = mbb(ref.problems)
    cfg = ref.solvers.SolverConfig(algorithm="pfbto_jacobi", max_iters=60, snapshot_every=20)
    got_states, want_states = [], []
    res = B.run(spec, cfg, sink=got_states.append)
    want = ref.solvers.run(spec, cfg, sink=want_states.append)
    assert res.reason == want.reason
    np.testing.assert_allclose(res.record.compliance, want.record.compliance, rtol=1e-9)
    np.testing.assert_allclose(res.record.dv_inf, want.record.dv_inf, rtol=1e-8, atol=1e-14)
    assert [s.iter for s in got_states] == [s.iter for s in want_states]
    for g, w in zip(got_states, want_states):
        np.testing.assert_allclose(g.v.values, w.v.values, rtol=0, atol=1e-9)
        np.testing.assert_allclose(g.u, w.u, rtol=0, atol=1e-9 * np.abs(w.u).max())


@pytest.mark.gpu
def test_l2_functions_with_reference_grid(ref, B):
    """apply_stiffness / element_energies / stiffness_diagonal / sensitivity /
    low_level_step on a reference GridModel (from the reference's resolve)."""
    spec = mbb(ref.problems, 37, 21)
    grid = ref.problems.resolve(spec)
    assert not isinstance(grid, B.GridModel)
    rng = np.random.default_rng(7)
    a = rng.uniform(1e-3, 1.0, grid.num_elements)
    u = rng.standard_normal(grid.num_dofs)
    y, yr = B.apply_stiffness(grid, a, u), ref.fea.apply_stiffness(grid, a, u)
    assert np.linalg.norm(y - yr) <= 1e-12 * np.linalg.norm(yr)
    np.testing.assert_allclose(B.element_energies(grid, u), ref.fea.element_energies(grid, u),
                               rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(B.stiffness_diagonal(grid, a), ref.fea.stiffness_diagonal(grid, a),
                               rtol=1e-13)
    vp = rng.uniform(0.1, 1.0, grid.num_elements)
    fs = ref.filtering.FilterSpec(7, 1.5)
    np.testing.assert_allclose(B.sensitivity(grid, vp, u, 3.0, fs),
                               ref.solvers.sensitivity(grid, vp, u, 3.0, fs), rtol=1e-13,
                               atol=1e-15)
    for algo in ("fbto", "pfbto_jacobi"):
        cfg = ref.solvers.SolverConfig(algorithm=algo)
        out = B.low_level_step(grid, a, u, cfg, 0.37)
        want = ref.solvers.low_level_step(grid, a, u, cfg, 0.37)
        np.testing.assert_allclose(out, want, rtol=0, atol=1e-12 * np.abs(want).max())
    # the device copy is cached per object and reused
    from paper_2204_06204_b200 import fea
    h = fea.grid_handle(grid)
    assert fea.grid_handle(grid) == h
    g2 = ref.problems.resolve(spec)
    assert fea.grid_handle(g2) != h


@pytest.mark.gpu
def test_integration_snippet_executes(ref, B, monkeypatch):
    """INTEGRATION.md §2, executed as written, gives the first record row of run()."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(import ctypes as C, numpy as np\n.*?)```", text, re.S).group(1)
    monkeypatch.chdir(ROOT)
    ns = {}
    exec(compile(code, "INTEGRATION.md#2", "exec"), ns)
    assert ns["rc"] == 0, ns["lib"].bsp_last_error()
    spec = ref.problems.catalog()["teaser"]
    res = B.run(spec, ref.solvers.SolverConfig(algorithm="cpfbto_krylov", max_iters=1))
    np.testing.assert_allclose(ns["rec"][0], res.record.compliance[0], rtol=1e-12)
    np.testing.assert_allclose(ns["rec"][3], res.record.volume[0], rtol=1e-12)
    ns["lib"].bsp_solver_destroy(ns["s"])
    ns["lib"].bsp_grid_destroy(ns["g"])


@pytest.mark.gpu
def test_config_struct_size_contract(B):
    """bsp_solver_config.struct_size: too small / too large is EINVAL; a
    caller struct that stops at max_batch gets the optional defaults."""
    import ctypes as C

    from paper_2204_06204_b200 import _native, fea
    from paper_2204_06204_b200.solvers import _prepare, config_c
    spec = B.problems.l_bracket(40)
    cfg = B.SolverConfig(algorithm="mg_pcg", max_iters=3)
    ws = _prepare(spec, cfg)
    c = config_c(ws, cfg, 4)
    v0 = np.ascontiguousarray(ws.v_init)
    act = np.ascontiguousarray(ws.active, dtype=np.uint8)
    h = C.c_void_p()
    lib = _native.load()
    for bad in (8, C.sizeof(_native.SolverConfigC) + 8):
        c.struct_size = bad
        rc = lib.bsp_solver_create(fea.grid_handle(ws.grid), C.byref(c), act.ctypes.data,
                                   v0.ctypes.data, C.byref(h))
        assert rc == _native.BSP_EINVAL and b"struct_size" in lib.bsp_last_error()
    # prefix up to max_batch: inner_steps/mg_* must come out as the defaults
    c.struct_size = _native.SolverConfigC.inner_steps.offset
    c.inner_steps, c.mg_omega, c.mg_nu = 99, -1.0, 0  # past struct_size: must be ignored
    _native.call("bsp_solver_create", fea.grid_handle(ws.grid), C.byref(c), act.ctypes.data,
                 v0.ctypes.data, C.byref(h))
    rec = np.zeros((4, 4))
    done, st = C.c_int(), C.c_int()
    alphas = np.array([cfg.step_size(k) for k in (1, 2, 3)])
    _native.call("bsp_solver_run", h, 1, 3, alphas.ctypes.data, rec.ctypes.data, C.byref(done),
                 C.byref(st))
    lib.bsp_solver_destroy(h)
    want = B.run(spec, cfg)
    np.testing.assert_allclose(rec[:3, 0], want.record.compliance, rtol=1e-12)


@pytest.mark.gpu
def test_launch_window_and_sequence_checked(B):
    """bsp_solver_launch rejects iterations outside the staged step sizes or
    out of sequence (they would read stale alphas / replay the wrong graph)."""
    import ctypes as C

    from paper_2204_06204_b200 import _native
    from paper_2204_06204_b200.solvers import DeviceLoop, _prepare
    spec = B.problems.mbb_half_beam(32, 16)
    cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=10)
    loop = DeviceLoop(_prepare(spec, cfg), cfg, max_batch=4)
    lib = _native.load()
    al = np.array([cfg.step_size(k) for k in (1, 2, 3, 4)])
    assert lib.bsp_solver_set_alphas(loop._h, 2, 4, al.ctypes.data) == _native.BSP_EINVAL
    _native.call("bsp_solver_set_alphas", loop._h, 1, 2, al.ctypes.data)
    assert lib.bsp_solver_launch(loop._h, 2) == _native.BSP_EINVAL      # out of sequence
    _native.call("bsp_solver_launch", loop._h, 1)
    _native.call("bsp_solver_launch", loop._h, 2)
    assert lib.bsp_solver_launch(loop._h, 3) == _native.BSP_EINVAL      # past the window
    rec = np.zeros((4, 4))
    done, st = C.c_int(), C.c_int()
    _native.call("bsp_solver_finish", loop._h, 1, 2, rec.ctypes.data, C.byref(done), C.byref(st))
    assert done.value == 2 and st.value == 0
    d, s, rows = loop.run(3, [cfg.step_size(k) for k in (3, 4)])
    assert d == 2
    with pytest.raises(ValueError):
        loop.run(2, [cfg.step_size(2)])
