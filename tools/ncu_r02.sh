set -x
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --import-source on --clock-control none -k regex:k_faces_tcs -s 4 -c 1 -o gpurun_out/tcs_p3 python tools/which_kernels.py 48 3 > gpurun_out/ncu_tcs.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:k_volume_tc -s 1 -c 1 -o gpurun_out/voltc_p3 python tools/which_kernels.py 48 3 > gpurun_out/ncu_vol.log 2>&1
$NCU --set full --import-source on --clock-control none -k regex:k_faces_fast -s 3 -c 1 -o gpurun_out/ff_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-implicit --power-iters 5 > gpurun_out/ncu_ff.log 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(faces|volume|red|wall)" --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --power-iters 20 > gpurun_out/ncu_c5.log 2>&1
tail -3 gpurun_out/ncu_c5.log
ls -la gpurun_out
