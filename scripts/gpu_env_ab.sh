#!/bin/bash
# A/B an environment override on one bench config (alternating rounds).
# usage: gpu_env_ab.sh "bench args" "ENV=a" "ENV=b" ...
ARGS=$1; shift
for r in 1 2; do for ev in "$@"; do
  env $ev timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e $ARGS > gpurun_out/ab.json 2>gpurun_out/ab.err
  echo "$ev: $(python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']/1e6,2), 'M/s', round(d['roofline']['frac'],4))" 2>&1 | tail -1)"
done; done
