#!/bin/bash
O=gpurun_out/cert2; mkdir -p $O
run() { name=$1; shift; timeout 900 python bench.py "$@" > $O/$name.json 2> $O/$name.err; echo "$name rc=$?"; python -c "
import json;d=json.load(open('$O/$name.json'));e=d.get('e2e') or {};c=d.get('cpu_baseline') or {}
print('$name', round(d['value']/1e6,3),'M/s e2e',round((e.get('value') or 0)/1e6,3),'frac',round(d['roofline']['frac'],3),'sum',d['config'].get('summation'),'cpu',c.get('value'),c.get('kind'))"; }
run n2v22_lognormal --weights lognormal
FW_CERT=0 run n2v22_lognormal_ordered --weights lognormal --nq 524288 --no-cpu-baseline
run n2v22_a3b07 --a 3 --b 0.7 --no-cpu-baseline
FW_CERT=0 run n2v22_a3b07_ordered --a 3 --b 0.7 --nq 524288 --no-cpu-baseline
run dw22_lognormal --app deepwalk --weights lognormal --no-cpu-baseline
run dw22 --app deepwalk --no-cpu-baseline
run dw22_lognormal_dprs --app deepwalk --weights lognormal --sampler dprs --no-cpu-baseline
