"""Generate golden input/output vectors from the REAL reference package.

Run in the builder container (the only place `/root/reference` exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes `tests/golden/*.npz`.  The fixtures are committed; the GPU box and the
CPU test suite read only the fixtures, never `/root/reference`.
Every case is seeded (`np.random.default_rng`) so the script is reproducible.
"""
from __future__ import annotations

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from bisimp import fea, filtering, projection, solvers  # noqa: E402
from bisimp.problems import ProblemSpec, catalog, resolve  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def cantilever_grid(nx, ny, nu=0.3):
    """Left edge clamped, unit downward load at right mid-height node (tests/oracles.py:14-35)."""
    n = 2 * (nx + 1) * (ny + 1)
    fixed = np.zeros(n, dtype=bool)
    for y in range(ny + 1):
        fixed[2 * y * (nx + 1)] = fixed[2 * y * (nx + 1) + 1] = True
    load = np.zeros(n)
    load[2 * ((ny // 2) * (nx + 1) + nx) + 1] = -1.0
    return fea.GridModel(nx=nx, ny=ny, ke=fea.element_stiffness(fea.Material(1.0, nu)),
                         fixed_dofs=fixed, load=load)


def random_fixture_grid(nx, ny, rng):
    n = 2 * (nx + 1) * (ny + 1)
    fixed = rng.uniform(size=n) < 0.15
    fixed[:3] = True
    load = rng.standard_normal(n)
    load[fixed] = 0.0
    return fea.GridModel(nx=nx, ny=ny, ke=fea.element_stiffness(fea.Material()),
                         fixed_dofs=fixed, load=load)


def grid_arrays(prefix, g, store):
    store[f"{prefix}_nx"] = g.nx
    store[f"{prefix}_ny"] = g.ny
    store[f"{prefix}_ke"] = g.ke
    store[f"{prefix}_fixed"] = g.fixed_dofs
    store[f"{prefix}_load"] = g.load


def make_fea():
    rng = np.random.default_rng(1000)
    s = {}
    for nu in (0.0, 0.2, 0.3, 0.45):
        s[f"ke_nu{int(nu * 100)}"] = fea.element_stiffness(fea.Material(1.0, nu))
    grids = {
        "g2x1": cantilever_grid(2, 1),
        "g3x2": cantilever_grid(3, 2),
        "g1x1": cantilever_grid(1, 1),
        "g7x5r": random_fixture_grid(7, 5, rng),
        "g16x12": cantilever_grid(16, 12),
        "g33x17r": random_fixture_grid(33, 17, rng),
        "g64x32": cantilever_grid(64, 32),
        "g40x70n45": cantilever_grid(40, 70, nu=0.45),
    }
    names = sorted(grids)
    s["grids"] = np.array(names)
    for name in names:
        g = grids[name]
        grid_arrays(name, g, s)
        a = rng.uniform(1e-3, 1.0, g.num_elements)
        u = rng.standard_normal(g.num_dofs)
        s[f"{name}_a"] = a
        s[f"{name}_u"] = u
        s[f"{name}_Ku"] = fea.apply_stiffness(g, a, u)
        s[f"{name}_diag"] = fea.stiffness_diagonal(g, a)
        s[f"{name}_energies"] = fea.element_energies(g, u)
        s[f"{name}_compliance"] = fea.compliance_energy(g, a, u)
        # near-equilibrium u: cancellation-heavy matvec input
        if g.num_dofs <= 5000:
            ue = fea.exact_solve(g, a, 1e-12) if np.any(g.load) else np.zeros(g.num_dofs)
            s[f"{name}_ueq"] = ue
            s[f"{name}_Kueq"] = fea.apply_stiffness(g, a, ue)
        s[f"{name}_rho50"] = fea.estimate_rho_max(g, a, 50, seed=3).rho_max
    np.savez_compressed(os.path.join(OUT, "fea.npz"), **s)


def make_filter():
    rng = np.random.default_rng(2000)
    s = {}
    cases = [(9, 6, 5, 1.2), (15, 11, 7, 1.5), (12, 9, 7, 1.5), (1, 1, 7, 1.5),
             (2, 3, 7, 1.5), (33, 17, 9, 4.0), (5, 4, 1, 1.0), (64, 48, 7, 1.5),
             (100, 3, 11, 2.5), (4, 50, 3, 0.7)]
    for i, (nx, ny, size, sigma) in enumerate(cases):
        spec = filtering.FilterSpec(size, sigma)
        x = rng.uniform(0.1, 1.0, nx * ny)
        y = rng.standard_normal(nx * ny)
        s[f"c{i}_shape"] = np.array([nx, ny, size])
        s[f"c{i}_sigma"] = sigma
        s[f"c{i}_x"] = x
        s[f"c{i}_y"] = y
        s[f"c{i}_fwd"] = filtering.apply_filter(x, nx, ny, spec)
        s[f"c{i}_adj"] = filtering.apply_filter_adjoint(y, nx, ny, spec)
        s[f"c{i}_w"] = filtering.gaussian_weights(spec)
    s["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(OUT, "filter.npz"), **s)


def make_projection():
    rng = np.random.default_rng(3000)
    s = {}
    cases = []
    for _ in range(300):
        n = int(rng.integers(2, 40))
        lo = float(rng.uniform(0.01, 0.4))
        hi = float(rng.uniform(lo + 0.2, 2.0))
        budget = float(rng.uniform(n * lo, n * hi))
        v = rng.uniform(lo - 1.0, hi + 1.0, n)
        cases.append((v, lo, hi, budget))
    # ties at coincident breakpoints (tests/test_projection.py:63-69)
    cases.append((np.array([0.8, 0.8, 0.8, 0.8, 0.3, 0.3]), 0.1, 1.0, 2.0))
    cases.append((np.ones(3), 0.1, 1.0, 1.5))
    # large budget-active instances in the solver's regime
    for n in (1000, 50_000):
        v = rng.uniform(0.0, 1.3, n)
        cases.append((v, 0.1, 1.0, 0.4 * n))
    for i, (v, lo, hi, budget) in enumerate(cases):
        s[f"p{i}_v"] = v
        s[f"p{i}_b"] = np.array([lo, hi, budget])
        s[f"p{i}_out"] = projection.project_simplex(v, projection.SimplexBounds(lo, hi, budget))
    s["n_cases"] = len(cases)
    np.savez_compressed(os.path.join(OUT, "projection.npz"), **s)


def make_solver_pieces():
    rng = np.random.default_rng(4000)
    s = {}
    g = cantilever_grid(6, 5)
    grid_arrays("g", g, s)
    a = rng.uniform(0.001, 1.0, g.num_elements)
    s["a"] = a
    for j in range(3):
        b = rng.standard_normal(g.num_dofs)
        b[g.fixed_dofs] = 0.0
        s[f"b{j}"] = b
        for dim in (1, 3, 20):
            s[f"kry_b{j}_d{dim}"] = solvers.krylov_apply(g, a, b, dim)
    # exactness on the 2x1 grid (tests/test_solvers.py:153-159)
    g21 = cantilever_grid(2, 1)
    grid_arrays("g21", g21, s)
    s["kry21"] = solvers.krylov_apply(g21, np.full(2, 0.5), g21.load, 10)
    # larger Krylov case where the 21-column basis is ill conditioned
    gk = cantilever_grid(24, 16)
    grid_arrays("gk", gk, s)
    vk = rng.uniform(0.1, 1.0, gk.num_elements)
    ak = filtering.apply_filter(vk, 24, 16, filtering.FilterSpec()) ** 3
    uk = rng.standard_normal(gk.num_dofs) * 10
    uk[gk.fixed_dofs] = 0.0
    rk = fea.apply_stiffness(gk, ak, uk) - gk.load
    s["gk_a"], s["gk_u"], s["gk_r"] = ak, uk, rk
    s["gk_kry20"] = solvers.krylov_apply(gk, ak, rk, 20)
    # low-level steps
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        for algo in ("fbto", "pfbto_jacobi", "cpfbto_krylov"):
            cfg = solvers.SolverConfig(algorithm=algo)
            s[f"low_{algo}"] = solvers.low_level_step(gk, ak, uk, cfg, beta=0.37)
    # sensitivity on a few shapes
    for i, (nx, ny) in enumerate([(5, 4), (24, 16), (31, 7)]):
        gg = cantilever_grid(nx, ny)
        vp = rng.uniform(0.1, 1.0, nx * ny)
        u = rng.standard_normal(gg.num_dofs)
        s[f"sens{i}_shape"] = np.array([nx, ny])
        s[f"sens{i}_vp"] = vp
        s[f"sens{i}_u"] = u
        s[f"sens{i}_out"] = solvers.sensitivity(gg, vp, u, 3.0, filtering.FilterSpec())
    # high-level steps, with and without a passive region
    v = rng.uniform(0.1, 1.0, 200)
    gsn = rng.uniform(0.0, 2.0, 200)
    active = np.ones(200, dtype=bool)
    active[50:90] = False
    v[~active] = 0.1
    s["hl_v"], s["hl_g"], s["hl_active"] = v, gsn, active
    b1 = projection.SimplexBounds(0.1, 1.0, 0.4 * 200)
    b2 = projection.SimplexBounds(0.1, 1.0, 0.4 * 160)
    s["hl_out_all"] = solvers.high_level_step(v, gsn, 0.3, b1)
    s["hl_out_all_nomean"] = solvers.high_level_step(v, gsn, 0.3, b1, mean_projection=False)
    s["hl_out_act"] = solvers.high_level_step(v, gsn, 0.3, b2, active=active)
    np.savez_compressed(os.path.join(OUT, "solver_pieces.npz"), **s)


def spec_to_arrays(prefix, spec, store):
    grid = resolve(spec)
    store[f"{prefix}_fixed"] = grid.fixed_dofs
    store[f"{prefix}_load"] = grid.load
    store[f"{prefix}_passive"] = spec.passive_mask()
    store[f"{prefix}_shape"] = np.array([spec.nx, spec.ny])


MBB = dict(volume_fraction=0.5,
           fixtures=({"edge": "left", "dofs": "x"}, {"point": (1.0, 1.0), "dofs": "y"}),
           loads=({"edge": "top", "span": (0.0, 0.02), "fy": -1.0},))


def make_problems():
    s = {}
    cat = catalog()
    for name in sorted(cat):
        for sc in (1.0, 0.25, 0.1):
            spec = cat[name].scale(sc) if sc != 1.0 else cat[name]
            spec_to_arrays(f"{name}_{int(sc * 100)}", spec, s)
    spec_to_arrays("mbb440", ProblemSpec(nx=440, ny=250, **MBB), s)
    spec_to_arrays("lbr300", ProblemSpec(nx=300, ny=300, **{
        "volume_fraction": 0.5,
        "fixtures": ({"edge": "top", "span": (0.0, 0.4), "dofs": "xy"},),
        "loads": ({"edge": "right", "span": (0.6, 0.675), "fy": -1.0},),
        "passive": ({"rect": (0.4, 0.0, 1.0, 0.6)},)}), s)
    np.savez_compressed(os.path.join(OUT, "problems.npz"), **s)


def trajectory(name, spec, config, s, keep_state=True):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = solvers.run(spec, config)
    rec = res.record
    s[f"{name}_rec"] = np.array([rec.iters, rec.compliance, rec.residual_inf,
                                 rec.dv_inf, rec.volume]).T
    s[f"{name}_reason"] = res.reason
    s[f"{name}_cfg"] = np.array([config.algorithm, str(config.max_iters)])
    st = res.state
    if keep_state:
        s[f"{name}_u"] = st.u
        s[f"{name}_v"] = st.v.values
        s[f"{name}_vphys"] = st.v_phys
    else:
        s[f"{name}_vsum"] = float(st.v.values.sum())
        s[f"{name}_vphys_norm"] = float(np.linalg.norm(st.v_phys))
    s[f"{name}_iter"] = st.iter


def make_trajectories():
    s = {}
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        Cfg = solvers.SolverConfig
        small = ProblemSpec(nx=8, ny=8, volume_fraction=0.4,
                            fixtures=({"edge": "left", "dofs": "xy"},),
                            loads=({"point": (1.0, 0.5), "fy": -1.0},))
        cat = catalog()
        trajectory("fbto_small", small, Cfg(algorithm="fbto", max_iters=60), s)
        trajectory("pfbto_small", small, Cfg(algorithm="pfbto_jacobi", max_iters=120), s)
        trajectory("cpfbto_small", small, Cfg(algorithm="cpfbto_krylov", max_iters=30), s)
        trajectory("pfbto_lshape16", cat["lshape"].scale(0.1),
                   Cfg(algorithm="pfbto_jacobi", max_iters=300), s)
        trajectory("fbto_teaser32", cat["teaser"].scale(0.125),
                   Cfg(algorithm="fbto", max_iters=200), s)
        trajectory("pfbto_teaser64", cat["teaser"].scale(0.25),
                   Cfg(algorithm="pfbto_jacobi", max_iters=500), s)
        trajectory("cpfbto_teaser64", cat["teaser"].scale(0.25),
                   Cfg(algorithm="cpfbto_krylov", max_iters=5), s)
        trajectory("cpfbto_conv_cant", cat["cantilever"].scale(0.125),
                   Cfg(algorithm="cpfbto_krylov", max_iters=50_000), s, keep_state=True)
        # full-size configs: records only (C1 teaser cpfbto, C2 MBB pfbto, C3 L-bracket pfbto)
        trajectory("C1_cpfbto", cat["teaser"], Cfg(algorithm="cpfbto_krylov", max_iters=10), s,
                   keep_state=False)
        trajectory("C2_pfbto", ProblemSpec(nx=440, ny=250, **MBB),
                   Cfg(algorithm="pfbto_jacobi", max_iters=100), s, keep_state=False)
        trajectory("C3_pfbto", ProblemSpec(nx=300, ny=300, volume_fraction=0.5,
                                           fixtures=({"edge": "top", "span": (0.0, 0.4),
                                                      "dofs": "xy"},),
                                           loads=({"edge": "right", "span": (0.6, 0.675),
                                                   "fy": -1.0},),
                                           passive=({"rect": (0.4, 0.0, 1.0, 0.6)},)),
                   Cfg(algorithm="pfbto_jacobi", max_iters=50), s, keep_state=False)
    np.savez_compressed(os.path.join(OUT, "trajectories.npz"), **s)


C3_SPEC = dict(volume_fraction=0.5,
               fixtures=({"edge": "top", "span": (0.0, 0.4), "dofs": "xy"},),
               loads=({"edge": "right", "span": (0.6, 0.675), "fy": -1.0},),
               passive=({"rect": (0.4, 0.0, 1.0, 0.6)},))


def make_configs():
    """BASELINE configs as configured, at full size (VERDICT r01 "next" #1):
    C2 MBB 440x250 pfbto_jacobi for 1000 outer iterations and C3 L-bracket
    300x300 pfbto_jacobi for 500, each with the full record and the final
    per-element state (u, v, v_phys); C3 pgd_exact (the reference's SuperLU
    exact inversion, ~6.5 s per iteration here) for its first 30 iterations,
    the anchor for the GPU pgd_exact that grades the C3 MG-PCG endpoint."""
    s = {}
    Cfg = solvers.SolverConfig
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        trajectory("C2_pfbto1000", ProblemSpec(nx=440, ny=250, **MBB),
                   Cfg(algorithm="pfbto_jacobi", max_iters=1000), s)
        trajectory("C3_pfbto500", ProblemSpec(nx=300, ny=300, **C3_SPEC),
                   Cfg(algorithm="pfbto_jacobi", max_iters=500), s)
        trajectory("C3_pgd30", ProblemSpec(nx=300, ny=300, **C3_SPEC),
                   Cfg(algorithm="pgd_exact", max_iters=30), s)
    np.savez_compressed(os.path.join(OUT, "configs.npz"), **s)


def make_c3_endpoint():
    """C3 converged endpoints (VERDICT r01 "next" #1).  The reference's
    pgd_exact needs ~6.5 s per iteration here (SuperLU at 181k DOFs) and ~5000
    iterations at C3, so its endpoint is certified instead of recomputed:
    the GPU pgd_exact endpoint (tools/c3_endpoints.py, whose first 30
    iterations are pinned to the reference's at 3e-10 in configs.npz) is
    evaluated by the reference's own exact compliance (SuperLU, fea.py:230-275;
    test_acceptance.py:77-80).  The reference's cpfbto_krylov is run to
    convergence here (1405 iterations, ~5 min)."""
    spec = ProblemSpec(nx=300, ny=300, **C3_SPEC)
    grid = resolve(spec)

    def exact_compliance(v):
        a = filtering.apply_filter(v, spec.nx, spec.ny, spec.filter) ** spec.eta
        return 0.5 * float(grid.load @ fea.exact_solve(grid, a, 1e-10))

    gpu = np.load(os.path.join(os.path.dirname(OUT), "..", "gpurun_out", "c3_endpoints.npz"))
    s = {"pgd_v": gpu["pgd_exact_v"], "pgd_iter": gpu["pgd_exact_iter"],
         "pgd_exact_compliance_ref": exact_compliance(gpu["pgd_exact_v"])}
    v_uni = np.full(spec.num_elements, spec.v_lo)
    v_uni[~spec.passive_mask()] = spec.volume_fraction
    s["uniform_exact_compliance_ref"] = exact_compliance(v_uni)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        res = solvers.run(spec, solvers.SolverConfig(algorithm="cpfbto_krylov", max_iters=50_000))
    s["cpfbto_reason"] = res.reason
    s["cpfbto_iter"] = np.int64(res.state.iter)
    s["cpfbto_exact_compliance_ref"] = exact_compliance(res.state.v.values)
    np.savez_compressed(os.path.join(OUT, "c3_endpoint.npz"), **s)


def make_frames():
    """Density frames: the CLI's PGM bytes from the reference's own
    `outputs.write_snapshot` (outputs.py:21-30) and the service payload
    `v_phys.astype("<f4").tobytes()` (service/sessions.py:97) on a real
    teaser design plus adversarial values (pixel rounding ties, float32
    rounding ties, subnormals, overflow)."""
    import tempfile

    from bisimp import outputs

    s = {}
    res = solvers.run(catalog()["teaser"], solvers.SolverConfig(max_iters=20))
    vp = res.state.v_phys
    nx, ny = 128, 256
    s["design_v_phys"] = vp
    s["design_nx"], s["design_ny"] = np.int64(nx), np.int64(ny)
    rng = np.random.default_rng(11)
    j = np.arange(0, 511, dtype=np.float64)
    ties = np.clip(np.concatenate([j / 510.0, np.nextafter(j / 510.0, 2.0),
                                   np.nextafter(j / 510.0, -1.0), 1.0 - (j + 0.5) / 255.0]), 0.0, 1.0)
    px_vals = np.concatenate([ties, rng.uniform(0.0, 1.0, 4000), [0.0, 1.0, 0.5, 1e-300]])
    px_vals = px_vals[: (px_vals.size // 8) * 8 + 3]   # ragged length (not a multiple of 4)
    s["px_values"] = px_vals
    s["px_nx"], s["px_ny"] = np.int64(px_vals.size), np.int64(1)
    with tempfile.TemporaryDirectory() as d:
        for name, (v, w, h) in {"design": (vp, nx, ny), "px": (px_vals, px_vals.size, 1)}.items():
            path = os.path.join(d, f"{name}.pgm")
            outputs.write_snapshot(v, w, h, path)
            with open(path, "rb") as fh:
                s[f"{name}_pgm"] = np.frombuffer(fh.read(), dtype=np.uint8)
    f = np.float64
    half = [1.0 + 2.0 ** -24, 1.0 + 3 * 2.0 ** -24, 1.0 - 2.0 ** -25, 2.0 ** -149,
            2.0 ** -150, 1.5 * 2.0 ** -149, 1e-310, -1e-310, 1e-40, -1e-40, 3.4028235e38,
            3.4028236e38, 1e39, -1e39, np.inf, -np.inf, 0.0, -0.0]
    f32_vals = np.concatenate([np.array(half, dtype=f), vp[:2000],
                               rng.standard_normal(997) * 10.0 ** rng.integers(-40, 40, 997)])
    s["f32_values"] = f32_vals
    s["f32_payload"] = np.frombuffer(f32_vals.astype("<f4").tobytes(), dtype=np.uint8)
    s["design_payload"] = np.frombuffer(vp.astype("<f4").tobytes(), dtype=np.uint8)
    np.savez_compressed(os.path.join(OUT, "frames.npz"), **s)


def make_diagnostics():
    """diagnostics_projection_error (solvers.py:509-538) on reference states:
    the teaser at k=20 (no passive region) and the L-bracket (passive) at k=15,
    both with the iterate's u and with the exact solve."""
    s = {}
    cat = catalog()
    cases = {"teaser": (cat["teaser"].scale(0.25), 20),
             "lbracket": (ProblemSpec(nx=30, ny=30, volume_fraction=0.5,
                                      fixtures=({"edge": "top", "span": (0.0, 0.4),
                                                 "dofs": "xy"},),
                                      loads=({"edge": "right", "span": (0.6, 0.7),
                                              "fy": -1.0},),
                                      passive=({"rect": (0.4, 0.0, 1.0, 0.6)},)), 15),
             "small8": (ProblemSpec(nx=8, ny=8, volume_fraction=0.4,
                                    fixtures=({"edge": "left", "dofs": "xy"},),
                                    loads=({"point": (1.0, 0.5), "fy": -1.0},)), 10)}
    for name, (spec, k) in cases.items():
        cfg = solvers.SolverConfig(max_iters=k)
        st = solvers.run(spec, cfg).state
        s[f"{name}_v"], s[f"{name}_u"], s[f"{name}_k"] = st.v.values, st.u, np.int64(st.iter)
        s[f"{name}_err"] = solvers.diagnostics_projection_error(spec, st, cfg, k)
        try:  # the reference's SuperLU + refinement may miss its 1e-12 target (fea.py:272)
            s[f"{name}_err_exact"] = solvers.diagnostics_projection_error(spec, st, cfg, k,
                                                                          exact=True)
        except fea.LinearSolveError:
            s[f"{name}_err_exact"] = np.nan
    np.savez_compressed(os.path.join(OUT, "diagnostics.npz"), **s)


if __name__ == "__main__":
    which = sys.argv[1:] or ["fea", "filter", "projection", "solver_pieces", "problems",
                             "trajectories", "frames", "diagnostics", "configs"]
    for w in which:
        globals()[f"make_{w}"]()
        print("wrote", w)
