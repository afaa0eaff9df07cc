# Lightweight ncu metrics of the C5 (134M cells) pfbto iteration kernels:
# duration, instructions, DRAM bytes, issue activity.  One GPU.
#   bash tools/resid_ncu.sh TAG   -> gpurun_out/resid_TAG.csv
set -x
TAG=${1:-now}
mkdir -p gpurun_out
ncu --clock-control none --csv --page raw \
    --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread \
    -k 'regex:k_filter_fwd4|k_stiff3|k_filter_adj4|k_hl_' -s 101 -c 48 \
    python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/resid_$TAG.csv 2> gpurun_out/resid_$TAG.err
echo ncu_rc=$?
