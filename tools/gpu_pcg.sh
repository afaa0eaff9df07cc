# PCG vector kernels: tests, timing and an ncu capture of update/dir
set -x
mkdir -p gpurun_out
#timeout 900 python -m pytest tests/test_approx_inverse.py tests/test_distributed.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python tools/sharded_bench.py --world 1 --rank 0 --algo pcg_jacobi --steps 3 --warmup 3 --nx 8192 --ny 4096 2>&1 | tail -2
timeout 300 python tools/config_sweep.py C3 C4 --iters 10 2>&1 | grep -v "^{"
ncu --set full --clock-control none -k "regex:k_pcg_update|k_pcg_dir" -c 4 \
    -o gpurun_out/pcg_vec -f python tools/sharded_bench.py --world 1 --rank 0 --algo pcg_jacobi \
    --steps 1 --warmup 1 --nx 8192 --ny 4096 > gpurun_out/ncu_pcg.log 2>&1
