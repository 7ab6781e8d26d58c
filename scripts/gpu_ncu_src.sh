#!/bin/bash
# Source-attributed ncu capture of the Node2Vec walk kernel (bench workload, reduced query count)
NQ=${NQ:-262144}; TAG=${TAG:-n2v}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 \
  -o gpurun_out/prof_${TAG} python bench.py --steps 1 --warmup 0 --nq $NQ --no-cpu-baseline --no-e2e \
  > gpurun_out/ncu_${TAG}.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_${TAG}.log
