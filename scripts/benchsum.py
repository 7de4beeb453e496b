"""One-line summary of a bench.py JSON log.  python scripts/benchsum.py <log>"""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception:
        print(path, "ERR")
        continue
    r = d.get("roofline", {})
    print(d["config"]["workload"], f"value {d['value']:.3e} step {d['ms_per_step']:.3f}ms",
          f"frac {r.get('frac', 0):.3f} bound {r.get('bound')}",
          f"e2e {d.get('e2e', {}).get('value', 0):.3e}", f"kernel {r.get('kernel_ms', 0):.3f}ms")
