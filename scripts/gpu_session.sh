#!/bin/bash
# build, parity tests, bench + merge-ratio sweep
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for r in 0 2 4 8 32 100000; do
  FW_MERGE_RATIO=$r timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_mr$r.json 2>gpurun_out/bench_mr$r.err
  echo "ratio $r: $(python -c "import json;d=json.load(open('gpurun_out/bench_mr$r.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
done
