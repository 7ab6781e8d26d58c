#!/bin/bash
O=gpurun_out/qscan; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_certified.py tests/test_gpu_parity.py -x -q -m gpu -k "certified or golden or s16 or integer" > $O/pytest2.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest2.log
bash scripts/gpu_env_ab.sh "--a 3 --b 0.7" "FW_ISCAN=1" "FW_ISCAN=0"
bash scripts/gpu_env_ab.sh "--a 3 --b 0.7 --weights lognormal" "FW_ISCAN=1" "FW_ISCAN=0"
