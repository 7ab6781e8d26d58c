#!/bin/bash
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash scripts/gpu_abn.sh "" lib_v2.so
bash scripts/gpu_abn.sh "--app deepwalk --scale 16" lib_sorted.so lib_v2.so
bash scripts/gpu_abn.sh "--app deepwalk --scale 22" lib_sorted.so lib_v2.so
bash scripts/gpu_abn.sh "--app metapath --scale 24" lib_sorted.so lib_v2.so
bash scripts/gpu_abn.sh "--app ppr --scale 24 --queries hub --nq 2000000" lib_sorted.so lib_v2.so
