NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:k_faces_tcs -s 4 -c 1 -o gpurun_out/tcs_p3_fold python tools/face_bench.py 64 64 64 3 1 > gpurun_out/ncu_tcs2.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:k_volume_tc -s 1 -c 1 -o gpurun_out/voltc_p3b python tools/face_bench.py 64 64 64 3 1 > gpurun_out/ncu_vol2.log 2>&1
ls -la gpurun_out/*.ncu-rep | tail -2
