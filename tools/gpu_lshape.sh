for a in mg_pcg pcg_jacobi cpfbto_krylov mg_vcycle; do timeout 300 python tools/run_algo.py lshape64 $a 40000; done
timeout 600 python tools/run_algo.py lshape64 pgd_exact 5000
