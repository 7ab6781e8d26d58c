#!/bin/bash
# Round-end evidence: GPU suite, smoke, the reference arm, every config's bench line,
# launch list of the default bench.
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"; head -c 400 $O/bench_reference.json; echo
run() { name=$1; shift; timeout 1500 python bench.py "$@" > $O/bench_$name.json 2> $O/bench_$name.err; echo "$name rc=$?"; python -c "
import json;d=json.load(open('$O/bench_$name.json'));e=d.get('e2e') or {};c=d.get('cpu_baseline') or {};r=d['roofline']
print('$name', '%.4g'%d['value'],'e2e %.4g'%(e.get('value') or 0),'frac %.3f'%r['frac'],'dram_frac',r.get('dram_frac'),'cpu',c.get('value'), d['clocks'])"; }
run default
run dw16 --app deepwalk --scale 16
run dw22 --app deepwalk --scale 22
run mp24 --app metapath --scale 24
run ppr24_full --app ppr --scale 24 --queries hub
run n2v22_lognormal --weights lognormal
run s27_16m --scale 27 --nq 16777216 --no-cpu-baseline
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv python bench.py --steps 2 --warmup 1 > /dev/null 2>&1; echo "launches rc=$?"
