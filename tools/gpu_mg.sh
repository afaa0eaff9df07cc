# MG: tests, C3/C4 timing (fork / tail) and launch lists
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_approx_inverse.py -x -q -m gpu 2>&1 | tail -3
for f in 0 1; do
  BSP_MG_FORK=$f timeout 300 python tools/config_sweep.py C3 C4 --iters 20 2>&1 | grep -v "^{"
done
for c in C3; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python tools/config_sweep.py $c --iters 2 --warmup 2 > gpurun_out/ncu_$c.log 2>&1
done
