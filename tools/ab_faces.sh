# A/B of face-kernel builds / variants at one 3D size (tools/face_bench.py)
set -e
N=${N:-64}
for lib in paper_1403_1157_b200/libtaxisdg_b200.so paper_1403_1157_b200/lib_ab_*.so; do
  for var in 0 8192; do
    echo "== $lib variant $var"
    TDG_LIB=$lib python tools/face_bench.py $N $N $N 3 5 $var
  done
done
