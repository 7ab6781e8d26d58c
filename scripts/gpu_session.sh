#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
for m in 0 1; do
FW_N2V_MODE=$m timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_v9_m$m.json 2>gpurun_out/bench_v9_m$m.err
echo "n2v mode $m: $(python -c "import json;d=json.load(open('gpurun_out/bench_v9_m$m.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/prof_v9_300k python bench.py --nq 300000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_v9.log 2>&1; echo "ncu full rc=$?"
