# Source-level (SASS) instruction and stall attribution of one C5 pfbto
# kernel: one --set full capture with source, the source page exported as CSV
# on the box (the .ncu-rep stays there).
#   bash tools/src_ncu.sh TAG [KERNEL_REGEX]  -> gpurun_out/src_TAG_{sass,details}.csv
set -x
TAG=${1:-now}
KRX=${2:-'int\)1243>'}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$KRX" -s 1 -c 1 -o /tmp/src_$TAG -f \
    python tools/config_sweep.py C5 --iters 1 --warmup 2 > gpurun_out/src_$TAG.log 2>&1
echo ncu_rc=$?
ncu -i /tmp/src_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_sass.csv 2>&1
ncu -i /tmp/src_$TAG.ncu-rep --page details --csv > gpurun_out/src_${TAG}_details.csv 2>&1
ls -la gpurun_out/src_${TAG}_*
