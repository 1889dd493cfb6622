"""Print one summary line per bench JSON file (step time, value, per-kernel us)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    k = d.get("kernels", {})
    print(f"{f:40s} {d['config']['workload']:5s} {d['ms_per_step']:.3f} ms {d['value']:.3g} "
          + " ".join(f"{n}={v['us_per_step']:.0f}" for n, v in k.items())
          + f" frac={d.get('roofline', {}).get('frac', float('nan')):.3f}")
