"""One-line digest of bench.py JSON outputs: python tools/show_bench.py f1.json [f2.json ...]"""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    print(f"{d['config']['workload']}: {d['value']:.3g} rows/s  step {d['ms_per_step']:.3f} ms  "
          f"kernel {r.get('kernel_ms', float('nan')):.3f} ms  frac {r.get('frac', float('nan')):.3f}  "
          f"e2e {d.get('e2e', {}).get('value', float('nan')):.3g}")
