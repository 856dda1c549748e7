"""One-line summaries of bench.py JSON lines: python tools/bench_brief.py FILE..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    pk = r.get("per_kernel", {})
    e2e = d.get("e2e", {})
    rc = e2e.get("reference_call_shape", {})
    print(f"{f}: value {d['value']:.3e} {d['unit']}, {d['ms_per_step']:.2f} ms/step, frac {r.get('frac', 0):.3f}, "
          f"step_frac {r.get('step_frac', 0):.3f}, exec {r.get('step_executed_tflops', 0):.1f} TF")
    print("   " + ", ".join(f"{k}: {v['kernel']} {v['ms_per_application']:.2f} ms" for k, v in pk.items()))
    print(f"   e2e {e2e.get('value', 0):.3e} ({e2e.get('ms_per_step', 0):.1f} ms/step); "
          f"apply_f(numpy) {rc.get('ms_per_apply_f', 0):.0f} ms; cpu {d.get('cpu_baseline', {}).get('value', 0):.3e}; "
          f"clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
