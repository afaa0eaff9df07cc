"""Approximate inverses with no reference implementation (SURVEY §8(a')):
Jacobi-PCG-k, geometric-multigrid V-cycle and MG-preconditioned CG.

Graded as SURVEY §8(a') prescribes:
  * the CUDA path against the numpy restatement `oracle/approx_inverse_oracle.py`,
    per V-cycle and per PCG application, relative 2-norm error <= 1e-10
    (k <= 20 CG steps: the restatement differs in summation order only);
  * energy monotonicity 1/2 u.Ku - f.u at a fixed design (the pattern of the
    reference's tests/test_solvers.py:203-217); a residual contraction does
    NOT hold for CG and is not tested;
  * the converged MG-PCG design's exact compliance within 5% of pgd_exact
    (criterion 5 of the reference's tests/test_acceptance.py:198-226).
CPU tests pin the restatement itself (symmetry / definiteness of the V-cycle,
CG exactness at k = n, the coarse-mask rule)."""
import warnings

import numpy as np
import pytest

from oracle import approx_inverse_oracle as M
from oracle import bisimp_oracle as O

warnings.filterwarnings("ignore", message="decay exponent")

TOL = 1e-10


def oracle_grid(spec):
    return O.build_grid(spec.nx, spec.ny, spec.fixtures, spec.loads)


def specs():
    import paper_2204_06204_b200.problems as P
    return {
        "mbb": P.mbb_half_beam(60, 34),
        "lbracket": P.l_bracket(48),
        "ragged": P.ProblemSpec(nx=37, ny=5, volume_fraction=0.4,
                                fixtures=({"edge": "left", "dofs": "xy"},),
                                loads=({"point": (1.0, 0.5), "fy": -1.0},)),
    }


# ------------------------------------------------------------- CPU: oracle ---

def test_oracle_vcycle_symmetric_positive():
    g = oracle_grid(specs()["mbb"])
    rng = np.random.default_rng(0)
    a = rng.uniform(1e-3, 1.0, g.n_elem)
    lv = M.hierarchy(g.nx, g.ny, g.ke, g.fixed)
    acts = M.activations(lv, a)
    for nu in (1, 2):
        x, y = rng.standard_normal((2, g.n_dofs))
        x[g.fixed] = 0.0
        y[g.fixed] = 0.0
        vx, vy = M.vcycle(lv, acts, x, nu=nu), M.vcycle(lv, acts, y, nu=nu)
        assert abs(x @ vy - y @ vx) <= 1e-12 * abs(x @ vy)
        assert x @ vx > 0 and y @ vy > 0


def test_oracle_pcg_exact_at_full_dimension():
    spec = specs()["ragged"]
    import paper_2204_06204_b200.problems as P
    spec = P.ProblemSpec(nx=6, ny=3, volume_fraction=0.4, fixtures=spec.fixtures, loads=spec.loads)
    g = oracle_grid(spec)
    a = np.random.default_rng(1).uniform(0.1, 1.0, g.n_elem)
    K = M.dense_operator(M.Level(g.nx, g.ny, g.ke, g.fixed), a)
    f = np.where(g.fixed, 0.0, g.load)
    xs = np.linalg.solve(K, f)
    n_free = int((~g.fixed).sum())
    x = M.pcg(g, a, f, n_free)
    assert np.linalg.norm(x - xs) <= 1e-8 * np.linalg.norm(xs)


def test_oracle_coarse_mask_rule():
    g = oracle_grid(specs()["mbb"])
    lv = M.hierarchy(g.nx, g.ny, g.ke, g.fixed)
    assert [(l.nx, l.ny) for l in lv] == [(60, 34), (30, 17), (15, 9), (8, 5), (4, 3)]
    assert (lv[-1].nx + 1) * (lv[-1].ny + 1) <= M.COARSE_NODES
    for f, c in zip(lv[:-1], lv[1:]):
        F = f.fixed.reshape(f.ny + 1, f.nx + 1, 2)
        Cm = c.fixed.reshape(c.ny + 1, c.nx + 1, 2)
        assert Cm[:, 0, 0].all()  # the left edge stays clamped in x
        for Y in range(c.ny + 1):
            for X in range(c.nx + 1):
                ys = slice(max(0, 2 * Y - 1), min(f.ny, 2 * Y + 1) + 1)
                xs = slice(max(0, 2 * X - 1), min(f.nx, 2 * X + 1) + 1)
                assert (Cm[Y, X] == F[ys, xs].reshape(-1, 2).any(axis=0)).all()


# ------------------------------------------------------------ GPU: parity ---

@pytest.fixture(scope="module")
def B():
    import paper_2204_06204_b200 as B
    return B


def rel(x, y):
    return np.linalg.norm(np.asarray(x) - y) / max(np.linalg.norm(y), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mbb", "lbracket", "ragged"])
def test_mg_hierarchy_matches_oracle(B, name):
    spec = specs()[name]
    grid = B.resolve(spec)
    mg = B.Multigrid(grid)
    og = O.Grid.from_model(grid)
    lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed)
    assert mg.num_levels == len(lv)
    for l, ref in enumerate(lv):
        nx, ny, fixed = mg.level(l)
        assert (nx, ny) == (ref.nx, ref.ny)
        assert np.array_equal(fixed, ref.fixed)
    assert mg.coarse_dofs == lv[-1].grid.n_dofs


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mbb", "lbracket", "ragged"])
@pytest.mark.parametrize("nu", [1, 2])
def test_vcycle_matches_oracle(B, name, nu):
    spec = specs()[name]
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    rng = np.random.default_rng(2)
    a = rng.uniform(1e-3, 1.0, og.n_elem)
    b = rng.standard_normal(og.n_dofs)
    b[og.fixed] = 0.0
    mg = B.Multigrid(grid).setup(a)
    x = mg.vcycle(b, omega=0.6, nu=nu)
    lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed)
    ref = M.vcycle(lv, M.activations(lv, a), b, 0.6, nu)
    assert rel(x, ref) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["mbb", "lbracket", "ragged"])
@pytest.mark.parametrize("nu", [1, 2, 3])
def test_vcycle_tail_matches_multi_kernel(B, name, nu, monkeypatch):
    """The one-CTA coarse tail (BSP_MG_TAIL levels, csrc/mg.cu k_mg_tail) runs
    the same schedule and node-sum order as the per-level kernels; only FMA
    contraction inside the element algebra may differ (last-bit, measured
    <= 7e-16 relative)."""
    spec = specs()[name]
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    rng = np.random.default_rng(5)
    a = rng.uniform(1e-3, 1.0, og.n_elem)
    b = rng.standard_normal(og.n_dofs)
    b[og.fixed] = 0.0
    mg = B.Multigrid(grid).setup(a)
    out = {}
    for lim in ("0", "300", "600", "2048", str(10 ** 9)):  # off, partial, default, whole
        monkeypatch.setenv("BSP_MG_TAIL", lim)
        out[lim] = mg.vcycle(b, omega=0.6, nu=nu)
    for lim in ("300", "600", "2048", str(10 ** 9)):
        d = np.abs(out[lim] - out["0"]).max() / np.abs(out["0"]).max()
        assert d <= 1e-14, (lim, d)


@pytest.mark.gpu
@pytest.mark.parametrize("steps", [0, 1, 5, 20])
@pytest.mark.parametrize("precond", ["jacobi", "mg"])
def test_pcg_matches_oracle(B, steps, precond):
    spec = specs()["mbb"]
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    rng = np.random.default_rng(3)
    # a realistic design: filtered random densities, SIMP p = 3
    v = rng.uniform(0.1, 1.0, og.n_elem)
    a = O.filter_fwd(v, og.nx, og.ny) ** 3
    u = 0.1 * rng.standard_normal(og.n_dofs)
    u[og.fixed] = 0.0
    b = O.matvec(og, a, u) - og.load
    mg = B.Multigrid(grid) if precond == "mg" else None
    x = B.pcg_apply(grid, a, b, steps, mg)
    lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed) if precond == "mg" else None
    ref = M.pcg(og, a, b, steps, lv)
    assert rel(x, ref) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("precond", ["jacobi", "mg"])
def test_pcg_residual_history_matches_oracle(B, precond):
    # SURVEY §8(c) PCG contract: per-CG-step ||r_j|| within 1e-10 relative of
    # the numpy restatement for k <= 20 (r_j = b - K x_j with x_j the j-step
    # iterate from 0; every j is an independent pcg_apply call here)
    spec = specs()["lbracket"]
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    rng = np.random.default_rng(4)
    a = O.filter_fwd(rng.uniform(0.1, 1.0, og.n_elem), og.nx, og.ny) ** 3
    b = rng.standard_normal(og.n_dofs)
    b[og.fixed] = 0.0
    mg = B.Multigrid(grid) if precond == "mg" else None
    lv = M.hierarchy(og.nx, og.ny, og.ke, og.fixed) if precond == "mg" else None
    _, hist = M.pcg(og, a, b, 20, lv, history=True)
    floor = 1e-8 * hist[0]  # below it the residual is rounding noise (MG-PCG gets there)
    for j in (1, 2, 3, 5, 8, 13, 20):
        x = B.pcg_apply(grid, a, b, j, mg)
        r = b - O.matvec(og, a, x)
        r[og.fixed] = 0.0
        if hist[j] > floor:
            assert np.linalg.norm(r) == pytest.approx(hist[j], rel=1e-10), (precond, j)
        else:
            assert np.linalg.norm(r) <= floor, (precond, j)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["pcg_jacobi", "mg_vcycle", "mg_pcg"])
def test_low_level_step_matches_oracle(B, algo):
    spec = specs()["lbracket"]
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    rng = np.random.default_rng(4)
    a = O.filter_fwd(rng.uniform(0.1, 1.0, og.n_elem), og.nx, og.ny) ** 3
    u = 0.1 * rng.standard_normal(og.n_dofs)
    u[og.fixed] = 0.0
    cfg = B.SolverConfig(algorithm=algo, inner_steps=5 if algo != "mg_vcycle" else None)
    out = B.low_level_step(grid, a, u, cfg, 1.0)
    ref = M.low_level(og, a, u, algo, 1.0, steps=cfg.resolved_inner_steps(),
                      nu=cfg.resolved_mg_smooth())
    assert rel(out, ref) <= TOL


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["pcg_jacobi", "mg_vcycle", "mg_pcg"])
def test_energy_monotone_at_fixed_design(B, algo):
    # tests/test_solvers.py:203-217 pattern: repeated low-level steps at a fixed
    # design never increase the potential energy 1/2 u.Ku - f.u
    spec = specs()["mbb"]
    grid = B.resolve(spec)
    og = O.Grid.from_model(grid)
    a = O.filter_fwd(np.random.default_rng(5).uniform(0.1, 1.0, og.n_elem), og.nx, og.ny) ** 3
    cfg = B.SolverConfig(algorithm=algo)
    u = np.zeros(og.n_dofs)
    energies = []
    for _ in range(25):
        energies.append(0.5 * u @ O.matvec(og, a, u) - og.load @ u)
        u = B.low_level_step(grid, a, u, cfg, 1.0)
    e = np.array(energies)
    assert np.all(np.diff(e) <= 1e-12 * np.abs(e).max())
    assert e[-1] < e[1] < 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["pcg_jacobi", "mg_vcycle", "mg_pcg"])
def test_device_loop_trajectory_matches_oracle(B, algo):
    spec = specs()["lbracket"]
    cfg = B.SolverConfig(algorithm=algo, max_iters=40)
    res = B.run(spec, cfg)
    og = oracle_grid(spec)
    steps = cfg.resolved_inner_steps()
    beta, nu = cfg.resolved_beta(), cfg.resolved_mg_smooth()
    passive = spec.passive_mask()
    orc = O.run_loop(og, nx=spec.nx, ny=spec.ny, volume_fraction=spec.volume_fraction,
                     passive_mask=passive, algorithm=algo, max_iters=40,
                     low_level_fn=lambda g, a, u, r: M.low_level(g, a, u, algo, beta, r, steps,
                                                                 nu=nu))
    comp = np.array(res.record.compliance)
    ocomp = np.array([r[1] for r in orc["rows"]])
    assert len(comp) == len(ocomp) == 40
    # MG-PCG solves the lagged state accurately, and then the early outer
    # iterations at alpha0 = 0.25 swing over decades.  The reference's own
    # pgd_exact does the same on its L-shape: 2551, 9171, 69474, 16890, ...  The
    # swing amplifies summation-order differences about 3x per iteration
    # (measured on B200: 1.8e-12 at k=2, 7.8e-8 at k=10, 1e-4 at k=20).  So
    # mg_pcg is banded over its first 10 iterations, like the Krylov contract
    # of SURVEY §8(c).  Per application it matches the restatement to 1e-10
    # (above), and its endpoint is graded against pgd_exact (below).  The
    # stationary V-cycle amplifies more slowly (2.6e-9 at k=25, 4.5e-6 at
    # k=40); Jacobi-PCG-20 stays at rounding level over all 40 iterations.
    n = {"mg_pcg": 10, "mg_vcycle": 25, "pcg_jacobi": 40}[algo]
    assert np.all(np.abs(comp[:n] - ocomp[:n]) <= 1e-6 * np.abs(ocomp[:n]))
    if algo == "pcg_jacobi":
        vphys = O.filter_fwd(orc["last"][2], spec.nx, spec.ny)
        assert np.abs(res.state.v_phys - vphys).max() <= 1e-6


@pytest.fixture(scope="module")
def lshape_pgd(B):
    spec = B.catalog()["lshape"].scale(0.4)
    pgd = B.run(spec, B.SolverConfig(algorithm="pgd_exact", max_iters=50000))
    assert pgd.reason == "converged"
    return pgd


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["mg_pcg", "mg_vcycle", "pcg_jacobi"])
def test_converged_compliance_within_5pct_of_pgd(B, lshape_pgd, algo):
    # criterion 5 of the reference acceptance suite (test_acceptance.py:198-226)
    # on its L-shape (catalog()["lshape"].scale(0.4) = 64 x 64).  Measured on
    # B200: pgd_exact 777.80 (4324 iterations; the reference's 777.80);
    # mg_pcg (4 steps, 2+2 sweeps, beta 0.5) 801.4; mg_vcycle (1+1 sweeps)
    # 795.5; pcg_jacobi 760.49 (5003; SURVEY §8(a') scratch: 760.49 / 5003).
    # The endpoints are chaotic like CPFBTO's; the defaults were chosen on
    # this L-shape at 64^2, 160^2 and 300^2 together (solvers.py
    # _BETA_DEFAULTS; C3 itself: tests/test_configs_parity.py).
    spec = B.catalog()["lshape"].scale(0.4)
    res = B.run(spec, B.SolverConfig(algorithm=algo, max_iters=50000))
    assert res.reason == "converged"
    pgd = lshape_pgd
    grid = B.resolve(spec)

    def exact_compliance(v):
        vp = B.apply_filter(v, spec.nx, spec.ny, spec.filter)
        u = B.exact_solve(grid, vp ** spec.eta, 1e-10)
        return 0.5 * float(np.asarray(grid.load) @ u)

    c = exact_compliance(res.state.v.values)
    c_pgd = exact_compliance(pgd.state.v.values)
    assert abs(c - c_pgd) <= 0.05 * c_pgd, (c, c_pgd, res.state.iter, pgd.state.iter)
    v_uniform = np.full(spec.num_elements, spec.v_lo)
    v_uniform[~spec.passive_mask()] = spec.volume_fraction
    assert c <= 0.5 * exact_compliance(v_uniform)
