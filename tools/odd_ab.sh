# odd-nx matvec A/B (public apply_stiffness at 16383 x 8192 and the even size)
cp paper_2204_06204_b200/lib/libbisimp_b200.so /tmp/lib_orig.so
for v in Q0 Q3; do
  cp build/ab/lib$v.so paper_2204_06204_b200/lib/libbisimp_b200.so
  for nx in 16383 16384; do echo -n "$v: "; python tools/prof_matvec.py $nx 8192 5 0; done
done
cp /tmp/lib_orig.so paper_2204_06204_b200/lib/libbisimp_b200.so
