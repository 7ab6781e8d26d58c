#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for r in 32 4 1000; do
  FW_MERGE_RATIO=$r timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_hr$r.json 2>gpurun_out/bench_hr$r.err
  echo "ratio $r: $(python -c "import json;d=json.load(open('gpurun_out/bench_hr$r.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/prof_n2v_v3 python bench.py --nq 300000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_v3.log 2>&1; echo "ncu rc=$?"
