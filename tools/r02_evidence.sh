# r02 evidence on one B200: GPU tests, bench (+ reference arm), CG/MG
# per-kernel metrics.  Outputs stay small (CSV), copied back in gpurun_out/.
set -x
python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_ev.log 2>&1; echo pytest_rc=$?
python __graft_entry__.py smoke > gpurun_out/smoke_ev.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_ev.json 2> gpurun_out/bench_ev.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_ev.json 2> gpurun_out/bench_ref_ev.err; echo ref_rc=$?
timeout 600 ncu --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum -c 700 python tools/cg_roofline.py mg > gpurun_out/ncu_mg_c4_ev.csv 2> gpurun_out/ncu_mg_c4_ev.err; echo ncu_mg_rc=$?
timeout 600 ncu --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread -k regex:"k_pcg|k_stiff|k_diag" -c 8 python tools/cg_roofline.py cg > gpurun_out/ncu_cg_c5_ev.csv 2> gpurun_out/ncu_cg_c5_ev.err; echo ncu_cg_rc=$?
timeout 900 bash tools/resid_ncu.sh ev; echo resid_rc=$?
