#!/bin/bash
O=gpurun_out/cert3; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_certified.py tests/test_gpu_parity.py -x -q -m gpu -k "certified or golden or lognormal or s16 or integer" --durations=6 > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -9 $O/pytest.log
for args in "--app deepwalk --weights lognormal" "--app ppr --scale 24 --queries hub --weights lognormal --nq 2097152" "--app metapath --scale 24 --weights lognormal"; do
 for ev in FW_CERT=1 FW_CERT=0; do
  env $ev timeout 900 python bench.py $args --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/b.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/b.json'));print('$args $ev', '%.4g'%d['value'])"
 done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/ingest_launches.csv python scripts/bench_ingest.py --scales 24 --reps 2 > $O/ingest_ncu.jsonl 2>&1; echo "ingest ncu rc=$?"
