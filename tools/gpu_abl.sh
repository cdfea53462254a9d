#!/bin/bash
# A/B of library builds and knobs on one box: VARIANTS="label:lib.so:k=v,k=v ..." (lib under paper_1308_2166_b200/),
# each run REPS times, interleaved; optional pytest selection in TESTS (with -k expression in KEXPR)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if [ -n "$TESTS" ]; then
  if [ -n "$KEXPR" ]; then timeout 2400 python -m pytest -q -x $TESTS -k "$KEXPR" > gpurun_out/ab_tests.log 2>&1
  else timeout 2400 python -m pytest -q -x $TESTS > gpurun_out/ab_tests.log 2>&1; fi
  echo "tests rc=$?"; tail -3 gpurun_out/ab_tests.log
fi
CFG=${CFG:-C3}
for rep in $(seq 1 ${REPS:-1}); do
for v in $VARIANTS; do
  IFS=: read -r label lib kv <<< "$v"
  T=""; for x in ${kv//,/ }; do T="$T --tune $x"; done
  TC_LIB_PATH=$PWD/paper_1308_2166_b200/$lib timeout 900 python bench.py --config $CFG --no-e2e --no-cpu-baseline $EXTRA $T > gpurun_out/ab_$label.json 2> gpurun_out/ab_$label.err
  rc=$?
  python - "$label" "$rc" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    k = d["roofline"]["kernels"]
    print("%-8s ms/step %.4f " % (sys.argv[1], d["ms_per_step"]) + " ".join("%s=%.1f" % (n[2:], v["ms_per_launch"] * 1e3) for n, v in k.items() if v["ms_per_launch"] > 0.003))
except Exception as e:
    print(sys.argv[1], "rc", sys.argv[2], "failed", e)
PY
done
done
