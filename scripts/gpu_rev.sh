#!/bin/bash
# Reverse-search membership: parity under forced/default thresholds, then A/B.
O=gpurun_out/rev; mkdir -p $O
for rv in "1048576:1" "1:4"; do
  FW_REV=$rv timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -x -q -m gpu -k "golden or node2vec or n2v or s16 or integer" > $O/pytest_$rv.log 2>&1; echo "pytest FW_REV=$rv rc=$?"; tail -2 $O/pytest_$rv.log
done
bash scripts/gpu_env_ab.sh "" "FW_REV=0:1" "FW_REV=1:1" "FW_REV=1:4" "FW_REV=1:16"
