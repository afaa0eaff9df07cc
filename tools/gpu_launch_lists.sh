mkdir -p gpurun_out
for c in C1 C3 C4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python tools/config_sweep.py $c --iters 2 --warmup 2 > gpurun_out/ncu_$c.log 2>&1
done
