set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_solver_properties.py tests/test_approx_inverse.py tests/test_frames.py -x -q -m gpu 2>&1 | tail -2
bash tools/ab_c2.sh BSP_COND_FIX=0 BSP_COND_FIX=1
for f in 0 1; do BSP_COND_FIX=$f timeout 300 python tools/config_sweep.py C1 C2 C3 C5 --iters 20 2>&1 | grep -v "^{"; done
