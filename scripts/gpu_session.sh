#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
for v in base mb3 inl4 inl3; do
  lib=paper_2404_08364_b200/libflowwalk_$v.so; [ $v = base ] && lib=paper_2404_08364_b200/libflowwalk.so
  FW_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_v6_$v.json 2>gpurun_out/bench_v6_$v.err
  echo "n2v $v: $(python -c "import json;d=json.load(open('gpurun_out/bench_v6_$v.json'));print(d['value'], d['roofline']['frac'], d['ms_per_step'])")"
done
FW_LIB_PATH=$PWD/paper_2404_08364_b200/libflowwalk_inl4.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/prof_n2v_v6 python bench.py --nq 300000 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_v6.log 2>&1; echo "ncu rc=$?"
