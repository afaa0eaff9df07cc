set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_distributed.py tests/test_solver_properties.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/config_sweep.py C1 C2 --iters 50 2>&1 | grep -v "^{"
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_C1.csv python tools/config_sweep.py C1 --iters 2 --warmup 2 > gpurun_out/ncu_C1.log 2>&1
