"""Summarise bench JSON lines (tools/gpu_tune_c3.sh): step time, value and the per-kernel times."""
import json
import sys

for path in sys.argv[1:]:
    try:
        lines = [l for l in open(path) if l.startswith("{")]
        d = json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable:", e)
        continue
    r = d.get("roofline", {})
    ks = r.get("kernels", {})
    top = sorted(ks.items(), key=lambda kv: -kv[1]["ms_per_launch"] * kv[1]["launches"])
    print(f"{path}: {d['value']:.3e} edges/s  {d['ms_per_step']:.3f} ms/step  dominant {r.get('kernel')} "
          f"frac {r.get('frac') or 0:.3f}  whole {r.get('whole_step', {}).get('frac', 0):.3f}")
    print("    " + "  ".join(f"{k}={v['ms_per_launch'] * 1e3:.0f}us" for k, v in top))
