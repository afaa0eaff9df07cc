set -x
mkdir -p gpurun_out
BSP_FILTER4=5 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_distributed.py -x -q -m gpu 2>&1 | tail -2
for f in 2 5; do
BSP_FILTER4=$f ncu --set full --clock-control none -k 'regex:k_filter' -s 4 -c 2 \
    -o gpurun_out/c5_filt_$f -f python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/ncu_c5f_$f.log 2>&1
BSP_FILTER4=$f timeout 300 python tools/config_sweep.py C5 C2 --iters 50 2>&1 | grep -v "^{"
done
bash tools/ab_c2.sh BSP_FILTER4=2 BSP_FILTER4=5
