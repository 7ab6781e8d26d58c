#!/bin/bash
# GPU parity suite (all -m gpu tests), log under gpurun_out/$TAG.
O=gpurun_out/${TAG:-tests}; mkdir -p $O
timeout ${T:-1500} python -m pytest ${ARGS:-tests} -q -m gpu -x --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -40 $O/pytest_gpu.log
