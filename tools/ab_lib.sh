# A/B two builds of the library on the C2 bench: gpurun_out/libA.so vs libB.so
for i in 1 2 3; do
  for v in A B; do
    cp gpurun_out/lib$v.so paper_2204_06204_b200/lib/libbisimp_b200.so
    echo -n "$v: "; python bench.py --no-cpu --no-sweep --steps 2000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],5), round(d['ms_per_iter_hot'],5), round(d['e2e']['value'],5))"
  done
done
