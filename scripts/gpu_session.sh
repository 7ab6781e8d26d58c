#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
for cfg in "mp24:--app metapath --scale 24" "dw22:--app deepwalk --scale 22" "ppr24:--app ppr --scale 24 --queries hub --nq 2000000" "dw16:--app deepwalk --scale 16"; do
  n=${cfg%%:*}; a=${cfg#*:}
  timeout 900 python bench.py $a --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_$n.json 2>gpurun_out/bench_$n.err
  echo "$n: $(python -c "import json;d=json.load(open('gpurun_out/bench_$n.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
done
