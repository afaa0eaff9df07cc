# Warp-stall breakdown of the C5 pfbto iteration's big kernels (one GPU):
# --set full of the 3rd iteration's residual (k_stiff3<0,1243>), Jacobi step
# (k_stiff3<0,1156>) and adjoint filter, exported as CSV (raw + details).
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_stiff3|k_filter_adj4" \
    --launch-skip 104 -c 4 -o /tmp/stall_c5 -f \
    python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/stall_c5.log 2>&1
echo ncu_rc=$?
ncu -i /tmp/stall_c5.ncu-rep --page raw --csv > gpurun_out/stall_c5_raw.csv 2>/dev/null
ncu -i /tmp/stall_c5.ncu-rep --page details --csv > gpurun_out/stall_c5_details.csv 2>/dev/null
ncu -i /tmp/stall_c5.ncu-rep --page source --csv --print-source sass -k regex:"k_stiff3" --launch-count 1 > gpurun_out/stall_c5_sass.csv 2>/dev/null
echo export_rc=$?
ls -la gpurun_out
