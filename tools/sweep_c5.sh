#!/bin/bash
# C5 batch-size sweep (R-MAT scale 22, r = 2^22): one bench line per w (device-resident stream, graphs)
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for lw in ${LWS:-12 13 14 15 16 17 18 19 20 21 22 23 24}; do
  w=$((1 << lw)); st=$(( (1 << 26) / w )); [ $st -gt 200 ] && st=200; [ $st -lt 4 ] && st=4
  timeout 900 python bench.py --config C5 --w $w --steps $st --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sweep_$lw.json 2> gpurun_out/sweep_$lw.err
  echo "w=2^$lw rc=$?"
done
python tools/tune_summary.py gpurun_out/sweep_*.json
python - <<'PY'
import glob, json
rows = []
for p in sorted(glob.glob("gpurun_out/sweep_*.json"), key=lambda p: int(p.split("_")[-1].split(".")[0])):
    try:
        d = json.loads([l for l in open(p) if l.startswith("{")][-1])
    except Exception:
        continue
    r = d["roofline"]
    rows.append({"w": d["config"]["w"], "edges_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                 "estimator_updates_per_s": d["estimator_updates_per_s"], "dominant": r["kernel"],
                 "kernels_us": {k: round(v["ms_per_launch"] * 1e3, 1) for k, v in r["kernels"].items()},
                 "clocks": d.get("clocks")})
json.dump({"config": "C5: R-MAT scale 22 (64,153,382 edges), r = 2^22", "rows": rows}, open("gpurun_out/sweep_c5.json", "w"), indent=1)
PY
