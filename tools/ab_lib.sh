# Same-box A/B of library builds in build/ab/lib<V>.so (build/ab travels with
# the snapshot; gpurun_out does not):   bash tools/ab_lib.sh A B [configs...]
V1=${1:-A}; V2=${2:-B}; shift 2
CFGS=${@:-C5 C2}
cp paper_2204_06204_b200/lib/libbisimp_b200.so /tmp/lib_orig.so
for i in 1 2 3; do
  for v in $V1 $V2; do
    cp build/ab/lib$v.so paper_2204_06204_b200/lib/libbisimp_b200.so
    echo -n "$v: "; python tools/config_sweep.py $CFGS --iters 20 2>/dev/null | grep -o "^C[0-9a-z]*:\|[0-9.]* ms/iter" | tr '\n' ' '; echo
  done
done
cp /tmp/lib_orig.so paper_2204_06204_b200/lib/libbisimp_b200.so
