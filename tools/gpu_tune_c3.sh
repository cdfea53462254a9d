#!/bin/bash
# C3 geometry / estimator-pass variants (results are identical by construction; only time differs)
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --no-e2e --no-cpu-baseline --steps 14 --warmup 3"
$B > gpurun_out/tune_default.json 2>&1; echo default=$?
$B --tune split_kernels=1 > gpurun_out/tune_split.json 2>&1; echo split=$?
$B --tune vbucket_arcs=2048 > gpurun_out/tune_va2048.json 2>&1; echo va2048=$?
$B --tune vbucket_arcs=4096 > gpurun_out/tune_va4096.json 2>&1; echo va4096=$?
$B --tune vbucket_arcs=4096 --tune split_kernels=1 > gpurun_out/tune_va4096_split.json 2>&1; echo va4096s=$?
$B --config C2 --tune split_kernels=1 > gpurun_out/tune_c2_split.json 2>&1; echo c2split=$?
