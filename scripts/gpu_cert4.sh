#!/bin/bash
O=gpurun_out/cert4; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_certified.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for args in "--weights lognormal" "--a 3 --b 0.7" "--app deepwalk --weights lognormal" "--app ppr --scale 24 --queries hub --weights lognormal --nq 2097152" "--app metapath --scale 24 --weights lognormal"; do
 for ev in FW_CERT=1 FW_CERT=0; do
  env $ev timeout 900 python bench.py $args --steps 2 --warmup 1 --no-cpu-baseline --no-e2e ${NQ:+--nq $NQ} > $O/b.json 2>/dev/null
  python -c "import json;d=json.load(open('$O/b.json'));print('$args $ev', '%.4g'%d['value'])"
 done
done
