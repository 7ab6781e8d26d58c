#!/bin/bash
# Build a variant of the library with fw_walk.cu replaced by $1, output
# paper_2404_08364_b200/libflowwalk_$2.so (A/B runs with gpu_abn.sh).
set -e
D=$(mktemp -d); mkdir -p $D/p; cp -r paper_2404_08364_b200/csrc $D/p/; cp -r include $D/
cp "$1" $D/p/csrc/fw_walk.cu
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC -shared $XFLAGS -o paper_2404_08364_b200/libflowwalk_$2.so \
  $D/p/csrc/fw_api.cu $D/p/csrc/fw_walk.cu $D/p/csrc/fw_trials.cu $D/p/csrc/fw_ingest.cu
rm -rf $D
/usr/local/cuda/bin/cuobjdump -res-usage paper_2404_08364_b200/libflowwalk_$2.so 2>/dev/null | grep -A1 "walk_kernelILi2ELi1ELi1" | tail -1
