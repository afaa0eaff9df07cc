"""Bitwise run-to-run determinism of the device loop (every reduction is a
fixed-order tree; the forked iteration graph gives each branch its own
reduction scratch): two fresh loops on the same problem produce identical
records and designs, for the forked pfbto / cpfbto graphs, the fused
small-grid high-level step and the multigrid chain."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,algo,iters", [
    ("mbb440", "pfbto_jacobi", 300),   # C2: fused high-level step, forked graph
    ("mbb2400", "pfbto_jacobi", 60),   # 4.3M cells: the unfused adjoint + k_hl_write branch
    ("teaser", "cpfbto_krylov", 40),   # C1: Krylov chain beside the high-level branch
    ("lbracket", "mg_pcg", 40),        # passive region: unfused, multigrid chain
])
def test_device_loop_bitwise_reproducible(name, algo, iters):
    import paper_2204_06204_b200 as B
    from paper_2204_06204_b200 import solvers as S
    spec = {"mbb440": lambda: B.problems.mbb_half_beam(440, 250),
            "mbb2400": lambda: B.problems.mbb_half_beam(2400, 1800),
            "teaser": lambda: B.catalog()["teaser"],
            "lbracket": lambda: B.problems.l_bracket(96)}[name]()
    cfg = B.SolverConfig(algorithm=algo, max_iters=10 ** 9)
    outs = []
    for _ in range(2):
        ws = S._prepare(spec, cfg)
        loop = S.DeviceLoop(ws, cfg, max_batch=iters)
        done, status, rows = loop.run(1, [cfg.step_size(k) for k in range(1, iters + 1)])
        assert status == 0 and done == iters
        outs.append((rows.copy(), loop.read("v"), loop.read("u")))
        del loop
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
