"""The reference's seeded start vector on the device.

`np.random.default_rng(seed).standard_normal(n)` (fea.py:289-292,
solvers.py:352-355) restated as PCG64 + numpy's ziggurat:
  * CPU: the oracle restatement (oracle/rng_oracle.py), using the tables
    from the committed CUDA header, reproduces numpy bit for bit;
  * GPU: csrc/rng.cu reproduces numpy bit for bit, except that a tail sample
    (|x| > 3.65) may differ in its last bit (CUDA's log1p vs glibc's).
"""
import os

import numpy as np
import pytest

from oracle import rng_oracle as R

from conftest import ROOT

HEADER = os.path.join(ROOT, "paper_2204_06204_b200", "csrc", "ziggurat_tables.cuh")


@pytest.fixture(scope="module")
def tables():
    return R.read_tables(HEADER)


@pytest.mark.parametrize("seed", [0, 3, 2024])
def test_oracle_matches_numpy(tables, seed):
    n = 300_000
    assert np.array_equal(R.standard_normal(seed, n, tables),
                          np.random.default_rng(seed).standard_normal(n))


def test_oracle_pcg64_raw_and_advance():
    s, inc = R.pcg64_state(11)
    ref = np.random.PCG64(np.random.SeedSequence(11)).random_raw(2000)
    assert np.array_equal(R.pcg64_raw(s, inc, 2000), ref)
    for d in (1, 31, 32, 1000, 1999):
        assert np.array_equal(R.pcg64_raw(R.pcg64_advance(s, inc, d), inc, 2000 - d), ref[d:])


def test_header_records_numpy_version():
    text = open(HEADER).read()
    assert f'kNumpyVersion = "{np.__version__}"' in text, \
        "regenerate csrc/ziggurat_tables.cuh (tools/gen_ziggurat_tables.py) for this numpy"


# ------------------------------------------------------------------- GPU ---

def _check_stream(got, ref):
    got = np.asarray(got)
    diff = got != ref
    if diff.any():
        # only tail samples may differ, and only in the last bit
        assert np.all(np.abs(ref[diff]) > R.ZIG_R), ref[diff][:5]
        assert np.all(np.abs(got[diff] - ref[diff]) <= np.spacing(np.abs(ref[diff])))
    return int(diff.sum())


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 255, 256, 257, 4099, 1_000_000])
@pytest.mark.parametrize("seed", [0, 12345])
def test_device_standard_normal_matches_numpy(seed, n):
    from paper_2204_06204_b200 import fea
    got = fea.standard_normal(seed, n).cpu().numpy()
    assert got.shape == (n,)
    _check_stream(got, np.random.default_rng(seed).standard_normal(n))


@pytest.mark.gpu
def test_device_standard_normal_large():
    """30M normals (8k tail samples): bit-exact but for last-bit tail values."""
    from paper_2204_06204_b200 import fea
    n = 30_000_000
    got = fea.standard_normal(7, n).cpu().numpy()
    ref = np.random.default_rng(7).standard_normal(n)
    bad = _check_stream(got, ref)
    tails = int(np.sum(np.abs(ref) > R.ZIG_R))
    print(f"{n} normals: {n - bad} bit-identical, {bad} tail values off by 1 ulp of {tails} tails")
    assert bad <= tails


@pytest.mark.gpu
def test_device_start_vector_matches_reference_definition():
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import fea
    grid = B.resolve(B.problems.mbb_half_beam(440, 250))
    for seed in (0, 5):
        x = fea.start_vector(grid, seed).cpu().numpy()
        ref = R.start_vector(seed, np.asarray(grid.fixed_dofs))
        assert np.all(x[np.asarray(grid.fixed_dofs)] == 0.0)
        # the raw normals are identical; the norms differ by summation order
        np.testing.assert_allclose(x, ref, rtol=2e-15, atol=0)


@pytest.mark.gpu
def test_sparse_grid_equals_dense_grid():
    """The device grid scattered from resolve_sparse's lists equals the dense
    upload (masks, load, operator)."""
    import torch

    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import problems as P
    for spec in (P.mbb_half_beam(1638, 819), P.l_bracket(300), P.cantilever_square(1024)):
        dense, sparse = B.resolve(spec), P.resolve_device(spec)
        gen = torch.Generator(device="cuda").manual_seed(1)
        a = torch.rand(dense.num_elements, dtype=torch.float64, device="cuda", generator=gen)
        u = torch.randn(dense.num_dofs, dtype=torch.float64, device="cuda", generator=gen)
        assert torch.equal(B.apply_stiffness(dense, a, u), B.apply_stiffness(sparse, a, u))
        assert torch.equal(B.stiffness_diagonal(dense, a), B.stiffness_diagonal(sparse, a))
        r_d = B.fea.residual_reduce(dense, a, u)
        r_s = B.fea.residual_reduce(sparse, a, u)
        np.testing.assert_allclose(r_s[0].cpu().numpy(), r_d[0].cpu().numpy(), rtol=0,
                                   atol=1e-15 * float(r_d[0].abs().max()))


@pytest.mark.gpu
def test_c5_setup_on_device():
    """C5 (134M cells, 268M DOFs) set-up -- resolve, grid,
    beta's start vector and 50 power iterations -- without O(n) host work."""
    import time
    import warnings

    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import solvers as S
    warnings.filterwarnings("ignore", message="decay exponent")
    spec = B.problems.mbb_half_beam(16384, 8192)
    cfg = B.SolverConfig(algorithm="pfbto_jacobi", max_iters=1)
    t0 = time.perf_counter()
    ws = S._prepare(spec, cfg)
    loop = S.DeviceLoop(ws, cfg, max_batch=1)
    t1 = time.perf_counter()
    print(f"C5 set-up {t1 - t0:.2f} s (beta = {ws.beta:.6e})")
    assert isinstance(ws.grid, B.fea.SparseGridModel) and ws.grid._dense is None
    assert 0.0 < ws.beta < 1.0
    assert t1 - t0 < 3.0
    del loop
