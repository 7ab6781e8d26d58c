#!/bin/bash
# Round evidence: GPU parity suite, default bench line (cpu_baseline + e2e),
# launch list of the default bench command, one ncu --set full capture of the
# walk kernel on the bench workload (1M queries), and the other configs.
TAG=${TAG:-v17}
O=gpurun_out/prof_$TAG; mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 > $O/bench_under_launches.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o $O/full_n2v_1m \
  python bench.py --steps 1 --warmup 0 --nq 1048576 --no-cpu-baseline --no-e2e > $O/ncu_full_n2v_1m.json 2> $O/ncu_full.err; echo "ncu full rc=$?"
for cfg in "deepwalk --scale 16:dw16" "deepwalk --scale 22:dw22" "metapath --scale 24:mp24" "ppr --scale 24 --queries hub --nq 2000000:ppr24"; do
  args=${cfg%%:*}; name=${cfg##*:}
  timeout 900 python bench.py --app $args > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?"
done
timeout 1500 python bench.py --scale 27 --nq 16777216 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_s27_16Mq.json 2> $O/bench_s27.err; echo "s27 rc=$?"
