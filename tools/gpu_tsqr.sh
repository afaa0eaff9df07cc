set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k "regex:k_tsqr_merge" -c 1 -s 2 \
    -o gpurun_out/tsqr -f python tools/config_sweep.py C1 --iters 2 --warmup 1 > gpurun_out/ncu_tsqr.log 2>&1
