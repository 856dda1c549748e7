# e2e A/B over variant bits (alternating, 2 rounds): variant, e2e DoF-upd/s, e2e ms/step
for r in 1 2; do for v in ${@:-0 65536}; do python bench.py --variant $v --steps 20 --warmup 3 --no-implicit --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$v', e['value'], e['ms_per_step'])" >> gpurun_out/e2e_ab.txt; done; done
