#!/bin/bash
# Certified summation: parity (goldens in both orders, certified tests), then
# the log-normal Node2Vec bench with certification on and off (ordered kernels).
O=gpurun_out/cert; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_certified.py tests/test_gpu_parity.py -x -q -m gpu -k "certified or golden or lognormal or s16 or integer" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for ev in "FW_CERT=1" "FW_CERT=0"; do
  env $ev timeout 900 python bench.py --weights lognormal --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${NQ:+--nq $NQ} > $O/bench_$ev.json 2> $O/bench_$ev.err; echo "$ev rc=$?"
  python -c "import json;d=json.load(open('$O/bench_$ev.json'));print('$ev', round(d['value']/1e6,3),'M/s ms', round(d['ms_per_step'],1))"
done
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > $O/bench_default.json 2>/dev/null
python -c "import json;d=json.load(open('$O/bench_default.json'));print('default', round(d['value']/1e6,3),'M/s')"
