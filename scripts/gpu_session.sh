#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
timeout 900 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json
for cfg in "dw16:--app deepwalk --scale 16" "mp24:--app metapath --scale 24" "ppr24:--app ppr --scale 24 --queries hub --nq 2000000"; do
  n=${cfg%%:*}; a=${cfg#*:}
  timeout 900 python bench.py $a --steps 3 --warmup 3 --no-e2e --cpu-seconds 8 > gpurun_out/bench_$n.json 2>gpurun_out/bench_$n.err
  echo "$n: $(python -c "import json;d=json.load(open('gpurun_out/bench_$n.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'], d['cpu_baseline'] and d['cpu_baseline']['value'])")"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r01.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/prof_bench_r01 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_r01.log 2>&1; echo "ncu full rc=$?"
timeout 1200 python bench.py --scale 27 --nq 8000000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_s27.json 2>gpurun_out/bench_s27.err; echo "s27 rc=$?"; cat gpurun_out/bench_s27.json; tail -3 gpurun_out/bench_s27.err
