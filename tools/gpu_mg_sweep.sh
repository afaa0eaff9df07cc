for kw in "inner_steps=2" "inner_steps=3" "inner_steps=4" "inner_steps=2 mg_smooth=2" "inner_steps=1"; do
  timeout 300 python tools/run_algo.py lshape64 mg_pcg 40000 $kw
done
