# A/B of an env switch on the C2 bench (value, hot, e2e), alternating 3x
for i in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; env $v python bench.py --no-cpu --no-sweep --steps 2000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],5), round(d['ms_per_iter_hot'],5), round(d['e2e']['value'],5))"
  done
done
