#!/bin/bash
# ncu --set full of the headline walk kernel (Node2Vec s22, 1M queries) with
# source correlation; exports the SASS-level source page for local analysis.
TAG=${TAG:-ncu}; O=gpurun_out/$TAG; mkdir -p $O
NQ=${NQ:-1048576}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 \
  -o $O/full_n2v python bench.py --steps 1 --warmup 0 --nq $NQ --no-cpu-baseline --no-e2e $EXTRA \
  > $O/ncu_run.log 2>&1; echo "ncu rc=$?"
ncu -i $O/full_n2v.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2>/dev/null; echo "src rc=$?"
ncu -i $O/full_n2v.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null; echo "raw rc=$?"
ls -la $O
