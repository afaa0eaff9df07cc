# Source-level (CUDA line / SASS) instruction and stall attribution of the C5
# residual kernel k_stiff3<0, 1243>: one --set full capture with source, the
# source page exported as CSV on the box (the .ncu-rep stays there).
#   bash tools/src_ncu.sh TAG  -> gpurun_out/src_TAG_{cuda,sass}.csv
set -x
TAG=${1:-now}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:int\)1243>' -s 1 -c 1 -o /tmp/src_$TAG -f \
    python tools/config_sweep.py C5 --iters 1 --warmup 2 > gpurun_out/src_$TAG.log 2>&1
echo ncu_rc=$?
ncu -i /tmp/src_$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_${TAG}_cuda.csv 2>&1
ncu -i /tmp/src_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_sass.csv 2>&1
ncu -i /tmp/src_$TAG.ncu-rep --page details --csv > gpurun_out/src_${TAG}_details.csv 2>&1
ls -la gpurun_out/src_${TAG}_*
