set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k "regex:k_mg_coarse_factor" -c 1 \
    -o gpurun_out/mg_factor -f python tools/config_sweep.py C3 --iters 2 --warmup 1 > gpurun_out/ncu_tail.log 2>&1
