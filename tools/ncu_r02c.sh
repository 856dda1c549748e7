NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:k_faces_tcs -s 4 -c 1 -o gpurun_out/tcs_p3_r02 python tools/face_bench.py 64 64 64 3 1 > gpurun_out/ncu_tcs3.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:k_volume_tc -s 1 -c 1 -o gpurun_out/voltc_p3_r02 python tools/face_bench.py 64 64 64 3 1 > gpurun_out/ncu_vol3.log 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(faces|volume|wall)" --csv --log-file gpurun_out/launches_c5_r02.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --power-iters 20 > gpurun_out/ncu_c5b.log 2>&1
tail -2 gpurun_out/ncu_c5b.log
