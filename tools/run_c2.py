"""Run N outer iterations of the C2 workload on the device loop (ncu target).

    python tools/run_c2.py [iters] [algorithm]
"""
import os
import sys
import warnings

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
warnings.filterwarnings("ignore")
import paper_2204_06204_b200 as B  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
algo = sys.argv[2] if len(sys.argv) > 2 else "pfbto_jacobi"
res = B.run(B.problems.mbb_half_beam(), B.SolverConfig(algorithm=algo, max_iters=iters))
print(algo, res.reason, res.state.iter, res.record.compliance[-1])
