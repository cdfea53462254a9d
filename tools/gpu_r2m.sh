#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 14"
$B > gpurun_out/x_base.json 2>&1; echo base=$?
TC_LIB_PATH=paper_1308_2166_b200/libtc_pt4.so $B > gpurun_out/x_pt4.json 2>&1; echo pt4=$?
TC_LIB_PATH=paper_1308_2166_b200/libtc_pt3.so $B > gpurun_out/x_pt3.json 2>&1; echo pt3=$?
$B --tune vbucket_arcs=512 > gpurun_out/x_va512.json 2>&1; echo va512=$?
$B --tune vbucket_arcs=768 > gpurun_out/x_va768.json 2>&1; echo va768=$?
$B --tune vbucket_cap=1536 > gpurun_out/x_vc1536.json 2>&1; echo vc1536=$?
B2="timeout 600 python bench.py --config C2 --no-cpu-baseline --no-e2e --steps 28"
TC_LIB_PATH=paper_1308_2166_b200/libtc_pt4.so $B2 > gpurun_out/x_c2_pt4.json 2>&1; echo c2pt4=$?
$B2 > gpurun_out/x_c2_base.json 2>&1; echo c2base=$?
