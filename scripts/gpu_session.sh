#!/bin/bash
./scripts/mix_fma_check
FW_LIB_PATH=$PWD/paper_2404_08364_b200/libflowwalk_fma.so timeout 900 python -m pytest tests -x -q -m gpu -k "golden or s16" > gpurun_out/pytest_fma.log 2>&1; echo "pytest(fma lib) rc=$?"; tail -2 gpurun_out/pytest_fma.log
bash scripts/gpu_ab.sh paper_2404_08364_b200/libflowwalk_fma.so paper_2404_08364_b200/libflowwalk.so
