# r02 final evidence on one B200 (the round-end state): GPU tests, smoke,
# bench (+ reference arm), the bench launch list, one --set full capture of
# the roofline kernel, CG/MG/C5 per-kernel metrics.  Only CSV/text comes back
# in gpurun_out/ (the .ncu-rep files are exported and deleted on the box).
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/fin_pytest.log 2>&1; echo pytest_rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1; echo smoke_rc=$?
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err; echo ref_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 4000 \
    --log-file gpurun_out/fin_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-sweep --no-sharded \
    > gpurun_out/fin_ncu_launch.log 2>&1; echo launch_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stiff -s 2 -c 1 \
    -o /tmp/k_stiff3_134M -f python tools/prof_matvec.py 16384 8192 3 1 > gpurun_out/fin_ncu_full_mv.log 2>&1; echo full_rc=$?
ncu -i /tmp/k_stiff3_134M.ncu-rep --page raw --csv > gpurun_out/fin_k_stiff3_raw.csv 2>&1
ncu -i /tmp/k_stiff3_134M.ncu-rep --page details --csv > gpurun_out/fin_k_stiff3_details.csv 2>&1
rm -f /tmp/k_stiff3_134M.ncu-rep
timeout 600 ncu --clock-control none --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum -c 700 python tools/cg_roofline.py mg > gpurun_out/fin_ncu_mg_c4.csv 2> gpurun_out/fin_ncu_mg_c4.err; echo ncu_mg_rc=$?
timeout 600 ncu --clock-control none --csv --page raw --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread -k regex:"k_pcg|k_stiff|k_diag" -c 8 python tools/cg_roofline.py cg > gpurun_out/fin_ncu_cg_c5.csv 2> gpurun_out/fin_ncu_cg_c5.err; echo ncu_cg_rc=$?
timeout 900 bash tools/resid_ncu.sh fin; echo resid_rc=$?
tail -3 gpurun_out/fin_pytest.log; cat gpurun_out/fin_smoke.log | tail -2
