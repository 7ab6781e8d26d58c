#!/bin/bash
timeout 1200 python -m pytest tests -x -q -m gpu -k "golden or s16 or torchrun" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
bash scripts/gpu_ab.sh paper_2404_08364_b200/libflowwalk.so paper_2404_08364_b200/libflowwalk_prev.so
