for a in mg_pcg pcg_jacobi mg_vcycle; do timeout 300 python tools/run_algo.py lshape64 $a 40000; done
