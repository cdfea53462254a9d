#!/bin/bash
# A/B: SoA first partition (k_scatter 12 B/arc, k_split pass A 4 B/arc) vs HEAD, C3 and C5 w=2^24, then the
# GPU suite's split-path tests with the SoA library.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
B="timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 28"
for rep in 1 2; do
for v in base soa; do
  TC_LIB_PATH=paper_1308_2166_b200/libtc_$v.so $B > gpurun_out/soa_c3_${v}_$rep.json 2>gpurun_out/soa_c3_${v}_$rep.err; echo "c3 $v rc=$?"
done
done
for v in base soa; do
  TC_LIB_PATH=paper_1308_2166_b200/libtc_$v.so $B --config C5 --w 16777216 > gpurun_out/soa_c5_$v.json 2>gpurun_out/soa_c5_$v.err; echo "c5 $v rc=$?"
done
TC_LIB_PATH=paper_1308_2166_b200/libtc_soa.so timeout 1500 python -m pytest tests -m gpu -x -q -k "C3 or C5 or C4 or knobs or fuzz or checked or pair_filter or index_paths or hub or full_range" > gpurun_out/soa_tests.log 2>&1; echo "tests rc=$?"
