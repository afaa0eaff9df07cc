set -x
ncu --clock-control none --csv --page raw --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size -k "regex:k_tsqr|k_kry|k_stiff3|k_filter|k_hl" -c 40 python tools/config_sweep.py C5k --iters 1 --warmup 1 > gpurun_out/ncu_c5k2.csv 2> gpurun_out/ncu_c5k2.err
ncu --set full --clock-control none -k "regex:k_mg_|k_pcg_" -c 14 -o /tmp/mgfull -f python tools/cg_roofline.py mg > gpurun_out/mgfull.log 2>&1
ncu -i /tmp/mgfull.ncu-rep --page raw --csv > gpurun_out/mgfull_raw.csv 2>&1
rm -f /tmp/mgfull.ncu-rep
ls -la gpurun_out/ncu_c5k2.csv gpurun_out/mgfull_raw.csv
