# r02 evidence run on one B200 (outputs small enough to copy back: <= 64 MiB)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_r02a.json 2> gpurun_out/bench_ref_r02a.err; echo ref_rc=$?
timeout 600 python tools/cg_roofline.py both --json gpurun_out/cg_roofline_r02a.json > gpurun_out/cg_roofline_r02a.log 2>&1; echo cg_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_pcg|k_stiff|k_diag" -c 8 -o /tmp/ncu_cg_c5 -f python tools/cg_roofline.py cg > gpurun_out/ncu_cg_c5.log 2>&1; echo ncu_cg_rc=$?
ncu -i /tmp/ncu_cg_c5.ncu-rep --page raw --csv > gpurun_out/ncu_cg_c5_raw.csv 2>/dev/null; echo export_rc=$?
timeout 900 ncu --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum -c 700 python tools/cg_roofline.py mg > gpurun_out/ncu_mg_c4_metrics.csv 2> gpurun_out/ncu_mg_c4.err; echo ncu_mg_rc=$?
timeout 900 bash tools/resid_ncu.sh r02a; echo resid_rc=$?
ls -la gpurun_out
