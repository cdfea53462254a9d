for p in 1 0; do STEPS=90 BARGS="--tune l2_persist=$p" bash tools/gpu_ab.sh paper_1308_2166_b200/libtc_b200_pad.so paper_1308_2166_b200/libtc_b200_pad2.so | grep ms/step; done
