# ncu --set full of one C5 (134M cells) pfbto iteration's kernels on 1 GPU
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
    -k 'regex:k_filter_fwd|k_stiff|k_filter_adj|k_hl_' -s 119 -c 6 \
    -o gpurun_out/c5_iter -f python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/ncu_c5.log 2>&1
tail -5 gpurun_out/ncu_c5.log
