"""Parity at BASELINE.json's full sizes through size-independent properties.

The oracle cannot run a 134M-cell grid in test time, so at C5 (MBB
16384x8192, 134M cells, 268M DOFs) and C4 (cantilever 4096x4096) the CUDA path
is checked against identities the exact operators satisfy whatever the size:

* K(a) is linear and symmetric on the free DOFs, and u.K(a)u > 0 (fea.py:150-181);
* K(a)'s diagonal is what the matvec gives on unit vectors (fea.py:184-189);
* the filter is mass-normalised (C 1 = 1) and C^T is its adjoint,
  <C v, s> = <v, C^T s> (filtering.py:46-72);
* the simplex projection is feasible and idempotent (projection.py:50-91);
* the V-cycle is a symmetric operator and MG-PCG reduces the energy norm
  error monotonically (SURVEY §8(a'));
* the device frames agree with the host conversion through a checksum of
  checksums (service/sessions.py:97, outputs.py:27).

Inputs are generated on the device from fixed seeds (torch.Generator), so the
tests move no multi-GB host arrays.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import paper_2204_06204_b200 as B
    return B


@pytest.fixture(scope="module")
def c5(B):
    spec = B.problems.mbb_half_beam(16384, 8192)
    return spec, B.resolve(spec)


def _rand(torch, n, seed, lo=None, hi=None):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if lo is None:
        return torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    return lo + (hi - lo) * torch.rand(n, dtype=torch.float64, device="cuda", generator=g)


def _free(torch, grid):
    return torch.from_numpy(~np.asarray(grid.fixed_dofs, dtype=bool)).cuda()


def test_c5_matvec_linear_symmetric_positive(B, c5):
    import torch
    spec, grid = c5
    E, n = grid.num_elements, grid.num_dofs
    assert (E, n) == (134_217_728, 268_484_610)  # SURVEY §8 sizes table
    free = _free(torch, grid)
    a = _rand(torch, E, 1, 1e-3, 1.0)
    u = _rand(torch, n, 2) * free
    w = _rand(torch, n, 3) * free
    Ku = B.apply_stiffness(grid, a, u)
    Kw = B.apply_stiffness(grid, a, w)
    # symmetry on the free DOFs (the output is zero on fixed DOFs)
    uKw, wKu = float(torch.dot(u, Kw)), float(torch.dot(w, Ku))
    scale = float(torch.linalg.norm(u) * torch.linalg.norm(Kw))
    assert abs(uKw - wKu) <= 1e-12 * scale
    # linearity
    K3 = B.apply_stiffness(grid, a, u + 2.0 * w)
    err = float(torch.linalg.norm(K3 - (Ku + 2.0 * Kw)))
    assert err <= 1e-13 * float(torch.linalg.norm(Ku) + 2.0 * torch.linalg.norm(Kw))
    # positive energy, zero on fixed DOFs, K(a) 0 = 0
    assert float(torch.dot(u, Ku)) > 0.0
    assert float(torch.abs(Ku[~free]).max()) == 0.0
    assert float(torch.abs(B.apply_stiffness(grid, a, torch.zeros_like(u))).max()) == 0.0
    # compliance_energy is 1/2 u.Ku of the same operator
    c = B.compliance_energy(grid, a, u)
    assert c == pytest.approx(0.5 * float(torch.dot(u, Ku)), rel=1e-12)


def test_c5_diagonal_matches_unit_vectors(B, c5):
    import torch
    spec, grid = c5
    a = _rand(torch, grid.num_elements, 4, 1e-3, 1.0)
    d = B.stiffness_diagonal(grid, a)
    free = np.flatnonzero(~np.asarray(grid.fixed_dofs, dtype=bool))
    rng = np.random.default_rng(5)
    picks = np.concatenate([free[:3], free[-3:], rng.choice(free, 6, replace=False)])
    for j in picks:
        e = torch.zeros(grid.num_dofs, dtype=torch.float64, device="cuda")
        e[int(j)] = 1.0
        assert float(B.apply_stiffness(grid, a, e)[int(j)]) == pytest.approx(float(d[int(j)]),
                                                                            rel=1e-14)


def test_c5_filter_mass_and_adjoint(B, c5):
    import torch
    spec, grid = c5
    nx, ny = spec.nx, spec.ny
    ones = torch.ones(nx * ny, dtype=torch.float64, device="cuda")
    c1 = B.apply_filter(ones, nx, ny, spec.filter)
    assert float(torch.abs(c1 - 1.0).max()) <= 1e-15
    v = _rand(torch, nx * ny, 6, 0.1, 1.0)
    s = _rand(torch, nx * ny, 7)
    lhs = float(torch.dot(B.apply_filter(v, nx, ny, spec.filter), s))
    rhs = float(torch.dot(v, B.apply_filter_adjoint(s, nx, ny, spec.filter)))
    assert abs(lhs - rhs) <= 1e-12 * float(torch.linalg.norm(v) * torch.linalg.norm(s))


def test_c5_projection_feasible_idempotent(B, c5):
    import torch
    spec, grid = c5
    E = grid.num_elements
    bounds = B.SimplexBounds(0.1, 1.0, 0.5 * E)
    v = _rand(torch, E, 8, 0.0, 1.3)  # box sum above the budget: the lambda search runs
    p = B.project_simplex(v, bounds)
    assert float(p.min()) >= 0.1 and float(p.max()) <= 1.0
    assert abs(float(p.sum()) - 0.5 * E) <= 1e-7 * E
    p2 = B.project_simplex(p, bounds)
    assert float(torch.abs(p2 - p).max()) <= 1e-12


def test_c5_frames_checksum_of_checksums(B, c5):
    import torch
    from paper_2204_06204_b200.outputs import density_pixels, frame_payload
    spec, grid = c5
    E = grid.num_elements
    v = _rand(torch, E, 9, 0.0, 1.0)
    host = v.cpu().numpy()
    pay = np.frombuffer(frame_payload(v), dtype="<u4").reshape(-1, 1 << 20)
    ref = host.astype("<f4").view("<u4").reshape(-1, 1 << 20)
    # per-MiB-block checksums, then the checksum of those
    np.testing.assert_array_equal(pay.sum(axis=1, dtype=np.uint64), ref.sum(axis=1, dtype=np.uint64))
    px = density_pixels(v).cpu().numpy().reshape(-1, 1 << 20)
    rpx = np.floor(255.0 * (1.0 - host) + 0.5).astype(np.uint8).reshape(-1, 1 << 20)
    np.testing.assert_array_equal(px.sum(axis=1, dtype=np.uint64), rpx.sum(axis=1, dtype=np.uint64))
    assert int(px.sum(dtype=np.uint64)) == int(rpx.sum(dtype=np.uint64))


def test_c4_vcycle_symmetric_and_pcg_energy_monotone(B):
    import torch
    spec = B.problems.cantilever_square(4096)
    grid = B.resolve(spec)
    free = _free(torch, grid)
    a = _rand(torch, grid.num_elements, 10, 1e-3, 1.0)
    mg = B.Multigrid(grid).setup(a)
    x = _rand(torch, grid.num_dofs, 11) * free
    y = _rand(torch, grid.num_dofs, 12) * free
    xVy = float(torch.dot(x, mg.vcycle(y)))
    yVx = float(torch.dot(y, mg.vcycle(x)))
    assert abs(xVy - yVx) <= 1e-10 * abs(xVy)
    assert float(torch.dot(x, mg.vcycle(x))) > 0.0
    # MG-PCG from 0: the energy 1/2 x.Kx - b.x decreases with every CG step
    b = torch.from_numpy(np.asarray(grid.load)).cuda() * free
    energies = []
    for k in (1, 2, 4, 8):
        xk = B.pcg_apply(grid, a, b, k, multigrid=mg)
        energies.append(0.5 * float(torch.dot(xk, B.apply_stiffness(grid, a, xk)))
                        - float(torch.dot(b, xk)))
    assert all(e1 < e0 for e0, e1 in zip(energies, energies[1:])), energies
