# round-2 ncu evidence for the face-group / element-class kernels:
# full captures at 64^3 p = 3 (power-of-two cells: 12 face classes, 2
# element classes, like C5) and the C5 launch list with DRAM bytes
set -x
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:k_faces_tcg -c 1 -o gpurun_out/tcg_p3 python tools/face_bench.py 64 64 64 3 1 0 > gpurun_out/ncu_tcg.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:k_volume_tc -c 1 -o gpurun_out/volcls_p3 python tools/face_bench.py 64 64 64 3 1 0 > gpurun_out/ncu_volcls.log 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(faces|volume|red|wall)" --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --power-iters 20 > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_c5.log
ls -la gpurun_out
