L=paper_1403_1157_b200/libtaxisdg_b200.so
for r in 1 2; do for v in A B; do cp gpurun_out/ab/lib$v.so $L; echo "$v $(python tools/mgs_probe.py 2>/dev/null)" >> gpurun_out/ab.txt; done; done
