"""Pin the CPU oracle (oracle/bisimp_oracle.py) to golden vectors produced by
the real reference (tests/golden/make_golden.py).  CPU only."""
import os

import numpy as np
import pytest

from oracle import bisimp_oracle as O

from conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def grid_from(z, p):
    return O.Grid(int(z[f"{p}_nx"]), int(z[f"{p}_ny"]), z[f"{p}_ke"], z[f"{p}_fixed"],
                  z[f"{p}_load"])


def test_ke_matches_reference():
    z = load("fea.npz")
    for nu in (0.0, 0.2, 0.3, 0.45):
        np.testing.assert_allclose(O.q4_stiffness(1.0, nu), z[f"ke_nu{int(nu * 100)}"],
                                   rtol=0, atol=1e-15)


def test_fea_ops_match_reference():
    z = load("fea.npz")
    for name in z["grids"]:
        g = grid_from(z, name)
        a, u = z[f"{name}_a"], z[f"{name}_u"]
        scale = np.abs(z[f"{name}_Ku"]).max()
        np.testing.assert_allclose(O.matvec(g, a, u), z[f"{name}_Ku"], rtol=0,
                                   atol=1e-13 * scale)
        np.testing.assert_allclose(O.stiffness_diag(g, a), z[f"{name}_diag"], rtol=1e-14)
        np.testing.assert_allclose(O.energies(g, u), z[f"{name}_energies"], rtol=1e-13,
                                   atol=1e-15)
        c = 0.5 * float(u @ O.matvec(g, a, u))
        assert abs(c - float(z[f"{name}_compliance"])) <= 1e-12 * abs(c)
        if f"{name}_ueq" in z:
            ku = O.matvec(g, a, z[f"{name}_ueq"])
            ref = z[f"{name}_Kueq"]
            assert np.linalg.norm(ku - ref) <= 1e-10 * max(np.linalg.norm(ref), 1e-300) + 1e-14
        rho = O.power_rho(g, a, 50, seed=3)
        assert abs(rho - float(z[f"{name}_rho50"])) <= 1e-12 * abs(rho)


def test_filter_matches_reference():
    z = load("filter.npz")
    for i in range(int(z["n_cases"])):
        nx, ny, size = (int(t) for t in z[f"c{i}_shape"])
        sigma = float(z[f"c{i}_sigma"])
        np.testing.assert_allclose(O.gauss_taps(size, sigma), z[f"c{i}_w"], rtol=1e-15)
        np.testing.assert_allclose(O.filter_fwd(z[f"c{i}_x"], nx, ny, size, sigma),
                                   z[f"c{i}_fwd"], rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(O.filter_adj(z[f"c{i}_y"], nx, ny, size, sigma),
                                   z[f"c{i}_adj"], rtol=1e-13, atol=1e-14)


def test_projection_matches_reference():
    z = load("projection.npz")
    for i in range(int(z["n_cases"])):
        lo, hi, budget = z[f"p{i}_b"]
        out = O.project(z[f"p{i}_v"], lo, hi, budget)
        np.testing.assert_allclose(out, z[f"p{i}_out"], rtol=0, atol=1e-12)


def test_solver_pieces_match_reference():
    z = load("solver_pieces.npz")
    g = grid_from(z, "g")
    a = z["a"]
    for j in range(3):
        b = z[f"b{j}"]
        for dim in (1, 3, 20):
            out = O.krylov(g, a, b, dim)
            ref = z[f"kry_b{j}_d{dim}"]
            # Krylov-LSQ is conditioning-limited; compare the achieved residuals
            r_o = np.linalg.norm(b - O.matvec(g, a, out))
            r_r = np.linalg.norm(b - O.matvec(g, a, ref))
            assert abs(r_o - r_r) <= 1e-6 * np.linalg.norm(b)
            if dim <= 3:
                np.testing.assert_allclose(out, ref, rtol=0, atol=1e-9 * np.abs(ref).max())
    g21 = grid_from(z, "g21")
    np.testing.assert_allclose(O.krylov(g21, np.full(2, 0.5), g21.load, 10), z["kry21"],
                               atol=1e-9)
    gk = grid_from(z, "gk")
    ak, uk, rk = z["gk_a"], z["gk_u"], z["gk_r"]
    np.testing.assert_allclose(O.matvec(gk, ak, uk) - gk.load, rk, atol=1e-12)
    out = O.krylov(gk, ak, rk, 20)
    r_o = np.linalg.norm(rk - O.matvec(gk, ak, out))
    r_r = np.linalg.norm(rk - O.matvec(gk, ak, z["gk_kry20"]))
    assert abs(r_o - r_r) <= 1e-6 * r_r + 1e-12
    for algo in ("fbto", "pfbto_jacobi"):
        np.testing.assert_allclose(O.low_level(gk, ak, uk, algo, 0.37), z[f"low_{algo}"],
                                   rtol=0, atol=1e-12 * np.abs(z[f"low_{algo}"]).max())
    for i in range(3):
        nx, ny = (int(t) for t in z[f"sens{i}_shape"])
        gg = O.build_grid(nx, ny, ({"edge": "left", "dofs": "xy"},),
                          ({"point": (1.0, 0.5), "fy": -1.0},))
        out = O.sensitivity(gg, z[f"sens{i}_vp"], z[f"sens{i}_u"], 3.0)
        np.testing.assert_allclose(out, z[f"sens{i}_out"], rtol=1e-12, atol=1e-14)
    v, gs, act = z["hl_v"], z["hl_g"], z["hl_active"]
    np.testing.assert_allclose(O.high_level(v, gs, 0.3, 0.1, 1.0, 80.0), z["hl_out_all"],
                               atol=1e-12)
    np.testing.assert_allclose(O.high_level(v, gs, 0.3, 0.1, 1.0, 80.0, mean_projection=False),
                               z["hl_out_all_nomean"], atol=1e-12)
    np.testing.assert_allclose(O.high_level(v, gs, 0.3, 0.1, 1.0, 64.0, active=act),
                               z["hl_out_act"], atol=1e-12)


def _trajectory_case(z, name):
    rec = z[f"{name}_rec"]
    return rec


TRAJ = [
    # name, spec kwargs builder, algorithm, tolerance on compliance / v
    ("fbto_small", "fbto", 1e-12),
    ("pfbto_small", "pfbto_jacobi", 1e-12),
    ("cpfbto_small", "cpfbto_krylov", 1e-6),
    ("pfbto_lshape16", "pfbto_jacobi", 1e-10),
    ("fbto_teaser32", "fbto", 1e-10),
]


def _spec_args(name):
    from paper_2204_06204_b200.problems import ProblemSpec, catalog
    cat = catalog()
    small = ProblemSpec(nx=8, ny=8, volume_fraction=0.4,
                        fixtures=({"edge": "left", "dofs": "xy"},),
                        loads=({"point": (1.0, 0.5), "fy": -1.0},))
    return {"fbto_small": small, "pfbto_small": small, "cpfbto_small": small,
            "pfbto_lshape16": cat["lshape"].scale(0.1),
            "fbto_teaser32": cat["teaser"].scale(0.125)}[name]


@pytest.mark.parametrize("name,algo,tol", TRAJ)
def test_oracle_trajectory_matches_reference(name, algo, tol):
    z = load("trajectories.npz")
    spec = _spec_args(name)
    g = O.build_grid(spec.nx, spec.ny, spec.fixtures, spec.loads)
    pm = O.passive_mask(spec.nx, spec.ny, [p["rect"] for p in spec.passive])
    rec = z[f"{name}_rec"]
    out = O.run_loop(g, nx=spec.nx, ny=spec.ny, volume_fraction=spec.volume_fraction,
                     passive_mask=pm, algorithm=algo, max_iters=int(rec[-1, 0]))
    rows = np.array(out["rows"])
    assert rows.shape == rec.shape
    if algo == "cpfbto_krylov":
        # Krylov-LSQ trajectories are chaotic: contract §8(c)
        np.testing.assert_allclose(rows[:5, 1], rec[:5, 1], rtol=1e-2, atol=1e-14)
        return
    np.testing.assert_allclose(rows[:, 1], rec[:, 1], rtol=tol, atol=1e-14)
    np.testing.assert_allclose(rows[:, 4], rec[:, 4], rtol=tol)
    k, u, v, vp, a = out["last"]
    np.testing.assert_allclose(v, z[f"{name}_v"], rtol=0, atol=tol)


def test_oracle_frames_match_reference():
    """PGM bytes from the reference's outputs.write_snapshot and the service's
    float32 payload (tests/golden/make_golden.py::make_frames)."""
    z = load("frames.npz")
    for name in ("design", "px"):
        v, nx, ny = z[f"{name}_v_phys"] if name == "design" else z["px_values"], \
            int(z[f"{name}_nx"]), int(z[f"{name}_ny"])
        assert O.pgm_bytes(v, nx, ny) == z[f"{name}_pgm"].tobytes()
    assert O.frame_payload(z["f32_values"]) == z["f32_payload"].tobytes()
    assert O.frame_payload(z["design_v_phys"]) == z["design_payload"].tobytes()
    with pytest.raises(ValueError):
        O.pgm_bytes(np.array([0.5, 1.5]), 2, 1)
    with pytest.raises(ValueError):
        O.pgm_bytes(np.array([0.5, 0.5]), 3, 1)
