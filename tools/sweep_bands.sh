# e2e sweep over element bands: bands, e2e DoF-upd/s, e2e ms/step, host issue ms/step
for b in ${@:-4 8 12}; do python bench.py --bands $b --steps 20 --warmup 3 --no-implicit 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$b', d['value'], e['value'], e['ms_per_step'], e['host_issue_ms_per_step'])" >> gpurun_out/bands.txt; done
