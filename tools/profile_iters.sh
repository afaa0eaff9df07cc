# per-kernel evidence for the iteration of each config
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
    -k 'regex:k_filter|k_stiff|k_hl_' -s 119 -c 6 \
    -o gpurun_out/c5_iter_r2 -f python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/ncu_c5.log 2>&1
for c in C1 C3 C4; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$c.csv python tools/config_sweep.py $c --iters 2 --warmup 2 > gpurun_out/ncu_$c.log 2>&1
done
ls -la gpurun_out
