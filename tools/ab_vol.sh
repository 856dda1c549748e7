# A/B of alternative library builds at one 3D size (tools/face_bench.py)
N=${N:-64}
K=${K:-3}
for lib in paper_1403_1157_b200/lib_ab_*.so; do
  echo "== $lib"
  TDG_LIB=$lib python tools/face_bench.py $N $N $N $K 5 0
done
