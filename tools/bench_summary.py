"""One line per bench JSON: config, value ms, device-resident ms, k_tail ms (A/B runs)."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e)
        continue
    km = {k: ms for k, _, ms in d.get("kernels_ms", [])}
    dr = d.get("device_resident", {}).get("ms")
    print(f"{d['config'].get('graph', '?'):8s} value_ms {d['ms_per_step']:.4f} device_ms {dr} "
          f"k_tail {km.get('k_tail')} e2e_ms {(d.get('e2e') or {}).get('ms')} kernels "
          + " ".join(f"{k}={v:.4f}" for k, v in km.items()))
