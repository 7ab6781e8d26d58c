#!/bin/bash
# A/B/n of library builds on one bench config (alternating rounds).
# usage: gpu_abn.sh "bench args" lib1.so lib2.so ...
ARGS=$1; shift
for r in 1 2; do for lib in "$@"; do
  FW_LIB_PATH=$PWD/paper_2404_08364_b200/$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$lib: $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']/1e6,2), 'M/s', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done; done
