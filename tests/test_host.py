"""CPU-only checks: the C-ABI library exports everything include/*.h declares,
and the host-side mirror of the reference API (config validation, problem
setup, control channel) behaves like the reference."""
import ctypes
import os
import re
import warnings

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

HEADER = os.path.join(ROOT, "include", "bisimp_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bsp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2204_06204_b200 import _native
    lib = ctypes.CDLL(_native.lib_path())
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes binding covers exactly the declared surface
    assert sorted(_native.SIGNATURES) == names
    assert lib.bsp_version() == 1


def test_library_is_sm100a_cubin():
    import subprocess
    from paper_2204_06204_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2204_06204_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", text, re.M), f


def test_compute_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200._native import NativeUnavailable
    g = B.resolve(B.catalog()["teaser"].scale(0.05))
    with pytest.raises(NativeUnavailable):
        B.apply_stiffness(g, np.ones(g.num_elements), np.zeros(g.num_dofs))


def test_solver_config_validation():
    import paper_2204_06204_b200 as B
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        c = B.SolverConfig()
    assert c.algorithm == "cpfbto_krylov" and c.krylov_dim == 20 and c.m == 0.75
    assert c.resolved_alpha0() == 0.25
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        assert B.SolverConfig(algorithm="fbto").resolved_alpha0() == 0.001
    with pytest.warns(UserWarning, match="boundary"):
        B.SolverConfig(m=0.75)
    for kw in [{"algorithm": "newton"}, {"alpha0": -1.0}, {"m": 0.5}, {"m": 1.0}, {"beta": 0.0},
               {"krylov_dim": 0}, {"eta": 0.5}, {"tol_dv": 0.0}]:
        with pytest.raises(ValueError):
            B.SolverConfig(**kw)
    c = B.SolverConfig(alpha0=0.8, m=0.8)
    assert c.step_size(1) == 0.8


def test_problem_setup_matches_reference():
    import paper_2204_06204_b200 as B
    z = np.load(os.path.join(GOLDEN, "problems.npz"))
    cat = B.catalog()
    for name in sorted(cat):
        for sc in (1.0, 0.25, 0.1):
            spec = cat[name].scale(sc) if sc != 1.0 else cat[name]
            p = f"{name}_{int(sc * 100)}"
            assert (spec.nx, spec.ny) == tuple(z[f"{p}_shape"])
            g = B.resolve(spec)
            np.testing.assert_array_equal(g.fixed_dofs, z[f"{p}_fixed"])
            np.testing.assert_array_equal(g.load, z[f"{p}_load"])
            np.testing.assert_array_equal(spec.passive_mask(), z[f"{p}_passive"])
    for p, spec in (("mbb440", B.problems.mbb_half_beam()), ("lbr300", B.problems.l_bracket(300))):
        g = B.resolve(spec)
        np.testing.assert_array_equal(g.fixed_dofs, z[f"{p}_fixed"])
        np.testing.assert_array_equal(g.load, z[f"{p}_load"])
        np.testing.assert_array_equal(spec.passive_mask(), z[f"{p}_passive"])


def test_element_stiffness_matches_reference():
    import paper_2204_06204_b200 as B
    z = np.load(os.path.join(GOLDEN, "fea.npz"))
    for nu in (0.0, 0.2, 0.3, 0.45):
        np.testing.assert_allclose(B.element_stiffness(B.Material(1.0, nu)),
                                   z[f"ke_nu{int(nu * 100)}"], rtol=0, atol=1e-15)
    from paper_2204_06204_b200.fea import element_dof_map
    from oracle.bisimp_oracle import element_dofs
    np.testing.assert_array_equal(element_dof_map(7, 5), element_dofs(7, 5))


def test_grid_and_spec_validation():
    import paper_2204_06204_b200 as B
    n = 12
    fixed = np.zeros(n, dtype=bool)
    fixed[:2] = True
    with pytest.raises(ValueError, match="3 DOFs"):
        B.GridModel(2, 1, B.element_stiffness(B.Material()), fixed, np.zeros(n))
    fixed[:4] = True
    load = np.zeros(n)
    load[0] = 1.0
    with pytest.raises(ValueError, match="zero on fixed"):
        B.GridModel(2, 1, B.element_stiffness(B.Material()), fixed, load)
    with pytest.raises(ValueError):
        B.ProblemSpec(nx=4, ny=4, volume_fraction=0.05, loads=({"point": (1, 1), "fy": -1},))
    with pytest.raises(ValueError):
        B.ProblemSpec(nx=4, ny=4, volume_fraction=0.4)
    with pytest.raises(ValueError):
        B.FilterSpec(4, 1.0)
    with pytest.raises(ValueError):
        B.SimplexBounds(0.1, 1.0, 0.1).validate(2)
    with pytest.raises(ValueError):
        B.Material(1.0, 0.5)


def test_run_control_channel():
    import paper_2204_06204_b200 as B
    c = B.RunControl()
    c.send(B.RunControl.PAUSE)
    c.send({"alpha0": 0.1})
    assert c.drain() == ["pause", {"alpha0": 0.1}]
    assert c.drain() == []


def test_gaussian_weights_match_reference():
    import paper_2204_06204_b200 as B
    z = np.load(os.path.join(GOLDEN, "filter.npz"))
    for i in range(int(z["n_cases"])):
        nx, ny, size = (int(t) for t in z[f"c{i}_shape"])
        np.testing.assert_array_equal(B.gaussian_weights(B.FilterSpec(size, float(z[f"c{i}_sigma"]))),
                                      z[f"c{i}_w"])


def test_bench_reference_arm_json_contract():
    # `bench.py --impl reference` runs the unmodified reference
    # (baseline/_ref; the oracle port when absent) on host cores: one JSON line
    # with the contract's keys, on the same metric/config as the B200 arm
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["value"] > 0.0 and line["higher_is_better"] is False
    want = "reference" if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "bisimp")) else "port"
    assert line["cpu_baseline"]["kind"] == want and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("C2")


@pytest.mark.gpu
def test_bench_b200_arm_json_contract():
    # the B200 arm's one JSON line: the driver's keys plus roofline, cpu_baseline,
    # e2e, clocks and gpu_launches (task contract)
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "200",
                          "--warmup", "3", "--no-sweep", "--cpu-seconds", "2"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.strip()]
    assert len(lines) == 1
    line = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert key in line, key
    assert line["steps"] == 200 and line["warmup"] == 3 and line["n_gpus"] == 1
    r = line["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0.5 < r["frac"] < 1.2
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] == 1
    e2e = line["e2e"]
    assert e2e["value"] > 0.0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] > 0 and {"sm_mhz", "sm_max_mhz", "reasons"} <= set(line["clocks"])


def test_resolve_sparse_matches_resolve():
    """problems.resolve_sparse (the O(boundary) set-up of large grids, SURVEY
    §8(f)2) gives resolve()'s fixed DOFs and load support exactly, and its
    load values to 2 ulps (the norm's summation order may differ)."""
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import problems as P
    specs = list(B.catalog().values()) + [P.mbb_half_beam(), P.l_bracket(300),
                                          P.cantilever_square(512), P.mbb_half_beam(1638, 819)]
    for spec in specs:
        g = B.resolve(spec)
        fixed, ldofs, lvals = P.resolve_sparse(spec)
        assert np.array_equal(np.nonzero(g.fixed_dofs)[0], fixed)
        assert np.array_equal(np.nonzero(g.load)[0], ldofs)
        assert np.all(np.abs(g.load[ldofs] - lvals) <= 2 * np.spacing(np.abs(lvals)))
        sg = P.resolve_device(spec)  # dense views materialise on demand
        assert np.array_equal(sg.fixed_dofs, g.fixed_dofs)
        assert np.allclose(sg.load, g.load, rtol=1e-15, atol=0)
        assert sg.num_dofs == g.num_dofs and np.array_equal(sg.ke, g.ke)
