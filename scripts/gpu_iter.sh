#!/bin/bash
# Iteration loop: GPU parity suite, then the headline bench (kernel value only)
# plus optional extra bench args sets separated by ';' in $EXTRA.
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open("gpurun_out/bench_iter.json"))
print("N2V s22:", round(d["value"]/1e6,2), "M steps/s, frac", round(d["roofline"]["frac"],4), "ms", round(d["ms_per_step"],1))
PY
IFS=';' read -ra SETS <<< "${EXTRA:-}"
for s in "${SETS[@]}"; do
  [ -z "$s" ] && continue
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $s > gpurun_out/bench_x.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_x.json'));print('$s', round(d['value']/1e6,2),'M/s frac',round(d['roofline']['frac'],4))"
done
