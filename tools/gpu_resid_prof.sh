mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k 'regex:k_stiff3' -s 6 -c 1 \
    -o gpurun_out/resid_c4 -f python tools/config_sweep.py C2 --iters 3 --warmup 3 > gpurun_out/ncu_resid.log 2>&1
