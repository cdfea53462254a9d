#!/bin/bash
# A/B on the bench workload: default vs. knob settings given in $AB (space-separated key=value lists, comma-joined)
# plus the parity tests named in $TESTS
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then timeout 1800 python -m pytest -q -x $TESTS > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log; fi
CFG=${CFG:-C3}
for ab in "" $AB; do
  T=""; for kv in ${ab//,/ }; do T="$T --tune $kv"; done
  timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline $T > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "[$ab] rc=$?"
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/ab.json").read().strip().splitlines()[-1])
k = d["roofline"]["kernels"]
print("  ms/step %.4f" % d["ms_per_step"], " ".join("%s=%.1f" % (n, v["ms_per_launch"] * 1e3) for n, v in k.items() if v["ms_per_launch"] > 0.003))
PY
done
