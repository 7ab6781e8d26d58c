#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
timeout 900 python bench.py --app metapath --scale 24 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_mp24b.json 2>gpurun_out/bench_mp24b.err
echo "mp24: $(python -c "import json;d=json.load(open('gpurun_out/bench_mp24b.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
timeout 600 python bench.py --app deepwalk --scale 22 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_dw22.json 2>gpurun_out/bench_dw22.err
echo "dw22: $(python -c "import json;d=json.load(open('gpurun_out/bench_dw22.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/prof_mp24 python bench.py --app metapath --scale 24 --nq 2000000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_mp24.log 2>&1; echo "ncu rc=$?"
