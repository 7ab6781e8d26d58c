#!/bin/bash
O=gpurun_out/ingest2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ingest.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 900 python scripts/bench_ingest.py --scales 22 24 > $O/ingest.jsonl 2> $O/ingest.err; echo "bench rc=$?"
python -c "
import json
for l in open('$O/ingest.jsonl'):
    d=json.loads(l); print(d['what'][:40], d.get('scale'), d.get('with_weights'), d.get('ms') or d.get('s'), d.get('reps_ms') or d.get('reps_s') or '', d.get('alg_gbs') or d.get('gbs'))"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python scripts/bench_ingest.py --scales 24 --reps 1 > /dev/null 2>&1; echo "ncu rc=$?"
