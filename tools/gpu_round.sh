# round evidence: GPU tests, smoke, default bench, reference arm, ncu launch list + full captures
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
( time timeout 900 python bench.py )  > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 4000 \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-sweep \
    > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_stiff -s 2 -c 1 \
    -o gpurun_out/k_stiff3_134M -f python tools/prof_matvec.py 16384 8192 3 1 > gpurun_out/ncu_full_mv.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k 'regex:k_filter|k_stiff|k_hl_' -s 119 -c 6 \
    -o gpurun_out/c5_iter -f python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/ncu_c5.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
grep -E "real" gpurun_out/bench.err || true
