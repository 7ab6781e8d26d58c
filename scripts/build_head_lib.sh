#!/bin/bash
# Build the committed HEAD's library as paper_2404_08364_b200/libflowwalk_h.so
# (for A/B runs against the working tree's libflowwalk.so).
set -e
D=$(mktemp -d); git archive HEAD paper_2404_08364_b200/csrc include | tar -x -C $D
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -shared -o paper_2404_08364_b200/libflowwalk_h.so \
  $D/paper_2404_08364_b200/csrc/fw_api.cu $D/paper_2404_08364_b200/csrc/fw_walk.cu $D/paper_2404_08364_b200/csrc/fw_trials.cu $D/paper_2404_08364_b200/csrc/fw_ingest.cu
rm -rf $D
