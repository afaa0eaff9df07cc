# A/B two builds on C5 and C2 (config_sweep): gpurun_out/libA.so vs libB.so
for i in 1 2 3; do
  for v in A B; do
    cp gpurun_out/lib$v.so paper_2204_06204_b200/lib/libbisimp_b200.so
    echo -n "$v: "; python tools/config_sweep.py C5 C2 --iters 30 2>/dev/null | grep -o "[0-9.]* ms/iter" | tr '\n' ' '; echo
  done
done
