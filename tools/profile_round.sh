# ncu evidence for profiles/: launch list of the bench command + full captures
# of the top kernels.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_short.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu \
    > gpurun_out/ncu_launch.log 2>&1
# full capture: the 134M-cell matvec (roofline kernel), solver variant
ncu --set full --clock-control none --import-source on -k regex:k_stiff -s 2 -c 1 \
    -o gpurun_out/k_stiff_134M -f python tools/prof_matvec.py 16384 8192 3 1 > gpurun_out/ncu_full_mv.log 2>&1
# full capture: one C2 iteration's kernels (after 40 iterations of warm-up launches)
ncu --set full --clock-control none --import-source on -k regex:'^k_' -s 400 -c 8 \
    -o gpurun_out/c2_iter -f python tools/run_c2.py 120 > gpurun_out/ncu_full_c2.log 2>&1
ls -la gpurun_out
