set -x
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 300 python tools/config_sweep.py C2 C5 --iters 30 2>&1 | grep -v "^{"
bash tools/ab_c2.sh BSP_X=1
ncu --set full --clock-control none -k 'regex:k_stiff3|k_filter' -s 6 -c 4 \
    -o gpurun_out/c5_apow -f python tools/config_sweep.py C5 --iters 3 --warmup 3 > gpurun_out/ncu_apow.log 2>&1
