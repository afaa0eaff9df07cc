for kw in "inner_steps=2" "inner_steps=3" "inner_steps=2 mg_omega=0.55" "inner_steps=2 mg_omega=0.65" "inner_steps=3 mg_omega=0.55" "inner_steps=4" "inner_steps=2 mg_smooth=1"; do
  timeout 300 python tools/run_algo.py lshape64 mg_pcg 50000 $kw
done
for kw in "inner_steps=20" "inner_steps=10"; do timeout 300 python tools/run_algo.py lshape64 pcg_jacobi 50000 $kw; done
