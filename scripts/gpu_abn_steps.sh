#!/bin/bash
# A/B/n of library builds on one bench config with a chosen step count.
# usage: gpu_abn_steps.sh STEPS "bench args" lib1.so lib2.so ...
S=$1; ARGS=$2; shift 2
for r in 1 2; do for lib in "$@"; do
  FW_LIB_PATH=$PWD/paper_2404_08364_b200/$lib timeout 600 python bench.py --steps $S --warmup 3 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$lib: $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']/1e6,2), 'M/s', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done; done
