#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python - > gpurun_out/l2fetch_default.txt <<'PY'
import torch, ctypes
torch.cuda.init()
lib = ctypes.CDLL("libcudart.so") if False else None
import cuda  # noqa
PY
for g in default 32 64 128; do
  if [ "$g" = default ]; then unset TC_L2_FETCH_BYTES; else export TC_L2_FETCH_BYTES=$g; fi
  python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 14 > gpurun_out/l2_$g.json 2> gpurun_out/l2_$g.err; echo "C3 $g rc=$?"
  python bench.py --config C2 --no-cpu-baseline --no-e2e --steps 28 > gpurun_out/l2c2_$g.json 2> gpurun_out/l2c2_$g.err; echo "C2 $g rc=$?"
done
