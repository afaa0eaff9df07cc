"""Run the masked Q4 matvec a few times at a given size (ncu / timing target).

    python tools/prof_matvec.py [nx] [ny] [launches] [inmask]

inmask=1 times the solver-internal variant (input known to be zero on fixed
DOFs); 0 (default) the public apply_stiffness path with input masking.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2204_06204_b200 as B  # noqa: E402
from paper_2204_06204_b200._native import call  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
launches = int(sys.argv[3]) if len(sys.argv) > 3 else 5
fn = "bsp_apply_stiffness_premasked" if len(sys.argv) > 4 and sys.argv[4] == "1" else "bsp_apply_stiffness"
g = B.resolve(B.problems.mbb_half_beam(nx, ny))
gen = torch.Generator(device="cuda").manual_seed(0)
a = torch.rand(g.num_elements, dtype=torch.float64, device="cuda", generator=gen) + 1e-3
u = torch.randn(g.num_dofs, dtype=torch.float64, device="cuda", generator=gen)
u[torch.from_numpy(g.fixed_dofs).cuda()] = 0.0
y = torch.empty_like(u)
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(launches):
    if i == launches - 1:
        ev[0].record(s)
    call(fn, g.native(), a.data_ptr(), u.data_ptr(), y.data_ptr(), s.cuda_stream)
ev[1].record(s)
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1])
n, E = g.num_dofs, g.num_elements
print(f"{fn} nx={nx} ny={ny} matvec {ms:.3f} ms  {(16 * n + 8 * E) / ms / 1e6:.0f} GB/s  {n / ms / 1e6:.1f} GDOF/s")
