# Same-box A/B in steady state (long warm-up: past the early lambda-search
# iterations):  bash tools/ab_steady.sh A B WARMUP ITERS [configs...]
V1=$1; V2=$2; W=$3; K=$4; shift 4
CFGS=${@:-C2}
cp paper_2204_06204_b200/lib/libbisimp_b200.so /tmp/lib_orig.so
for i in 1 2 3; do
  for v in $V1 $V2; do
    cp build/ab/lib$v.so paper_2204_06204_b200/lib/libbisimp_b200.so
    echo -n "$v: "; python tools/config_sweep.py $CFGS --iters $K --warmup $W 2>/dev/null | grep -o "^C[0-9a-z]*:\|[0-9.]* ms/iter" | tr '\n' ' '; echo
  done
done
cp /tmp/lib_orig.so paper_2204_06204_b200/lib/libbisimp_b200.so
