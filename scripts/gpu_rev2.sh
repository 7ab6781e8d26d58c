#!/bin/bash
O=gpurun_out/rev; mkdir -p $O
FW_REV=1048576:1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "golden or node2vec or n2v or s16 or integer" > $O/pytest_forced.log 2>&1; echo "pytest forced rc=$?"; tail -1 $O/pytest_forced.log
bash scripts/gpu_env_ab.sh "" "FW_REV=0:1" "FW_REV=1:2" "FW_REV=1:4" "FW_REV=1:16"
