#!/bin/bash
timeout 900 python -m pytest tests -x -q -m gpu -k "chi_square" > gpurun_out/pytest_chi.log 2>&1; echo "pytest chi rc=$?"; tail -2 gpurun_out/pytest_chi.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/prof_dw16 python bench.py --app deepwalk --scale 16 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_dw16.log 2>&1; echo "ncu rc=$?"
