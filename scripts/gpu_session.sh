#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
timeout 900 python bench.py > gpurun_out/bench_default.json 2>gpurun_out/bench_default.err; echo "bench rc=$?"; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 1500 python bench.py --scale 27 --nq 16000000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_s27.json 2>gpurun_out/bench_s27.err; echo "s27 rc=$?"; cat gpurun_out/bench_s27.json; tail -3 gpurun_out/bench_s27.err
