#!/bin/bash
# ncu --set full of the event mode's process and trigger kernels in the C5 w=4096 steady state (batch ~8000)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
PYTHONPATH=. timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k_ed_(process|trigger)" --launch-skip ${SKIP:-16000} --launch-count 4 \
  -o gpurun_out/ncu_ed_c5 python tools/dbg/ed_steady.py 4096 8000 20 > gpurun_out/ncu_ed.log 2>&1
echo ncu=$?; tail -3 gpurun_out/ncu_ed.log
