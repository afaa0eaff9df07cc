# same-box A/B of several library builds:  bash tools/ab_multi.sh "A B C" WARMUP ITERS configs...
VS=$1; W=$2; K=$3; shift 3
cp paper_2204_06204_b200/lib/libbisimp_b200.so /tmp/lib_orig.so
for i in 1 2; do
  for v in $VS; do
    cp build/ab/lib$v.so paper_2204_06204_b200/lib/libbisimp_b200.so
    echo -n "$v: "; python tools/config_sweep.py "$@" --iters $K --warmup $W 2>/dev/null | grep -o "^C[0-9a-z]*:\|[0-9.]* ms/iter" | tr '\n' ' '; echo
  done
done
cp /tmp/lib_orig.so paper_2204_06204_b200/lib/libbisimp_b200.so
