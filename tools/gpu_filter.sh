set -x
mkdir -p gpurun_out
ncu --set full --clock-control none -k 'regex:k_filter' -s 4 -c 2 \
    -o gpurun_out/c5_filt_2 -f python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/ncu_c5f_2.log 2>&1
timeout 300 python tools/config_sweep.py C5 C2 --iters 20 2>&1 | grep -v "^{"
