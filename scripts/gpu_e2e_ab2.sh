#!/bin/bash
for args in "" "--app deepwalk --scale 16"; do for lib in "$@"; do
  FW_LIB_PATH=$PWD/paper_2404_08364_b200/$lib timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $args > gpurun_out/e2e.json 2>/dev/null
  echo "$lib [$args]: $(python -c "import json;d=json.load(open('gpurun_out/e2e.json'));print(round(d['value']/1e6,2), 'e2e', round(d['e2e']['value']/1e6,2))" 2>&1 | tail -1)"
done; done
