#!/bin/bash
# Every BASELINE config at its own size (bench lines with cpu_baseline + e2e).
O=gpurun_out/cfg; mkdir -p $O
run() { name=$1; shift; timeout 1500 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; python -c "
import json;d=json.load(open('$O/$name.json'));e=d.get('e2e') or {};c=d.get('cpu_baseline') or {};r=d['roofline']
print('$name', '%.4g'%d['value'],'e2e %.4g'%(e.get('value') or 0),'frac %.3f'%r['frac'],'dram_frac',r.get('dram_frac'),'cpu',c.get('value'),c.get('kind'), d['clocks'])"; }
run default
run dw16 --app deepwalk --scale 16
run dw22 --app deepwalk --scale 22
run mp24 --app metapath --scale 24
run ppr24_full --app ppr --scale 24 --queries hub
run n2v22_lognormal --weights lognormal
run s27_16m --scale 27 --nq 16777216 --no-cpu-baseline
