# A/B of modal face kernel builds (64^3, p = 3 and p = 2) + parity of the last build
set -e
for lib in paper_1403_1157_b200/libtaxisdg_b200.so paper_1403_1157_b200/lib_ab_*.so; do
  for k in ${KS:-3 2}; do
    echo "== $lib p=$k"
    TDG_LIB=$lib python tools/face_bench.py 64 64 64 $k 5 | grep -E "faces|volume"
  done
done
