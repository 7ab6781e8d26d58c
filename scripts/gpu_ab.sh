#!/bin/bash
# A/B two builds of the walk library on the default bench (alternating)
A=${1:-paper_2404_08364_b200/libflowwalk.so}; B=${2:-paper_2404_08364_b200/libflowwalk_prev.so}
for r in 1 2; do for lib in $A $B; do
  FW_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$(basename $lib): $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']/1e6,2), 'M/s', round(d['roofline']['frac'],4))")"
done; done
