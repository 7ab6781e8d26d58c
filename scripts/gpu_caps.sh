#!/bin/bash
# ncu --set full captures (one walk_kernel launch each) of every BASELINE
# config's workload, with the bench line of the captured run (alg bytes).
O=gpurun_out/caps; mkdir -p $O
cap() { name=$1; shift
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o $O/$name \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e "$@" > $O/$name.json 2> $O/$name.err
  echo "$name ncu rc=$?"; }
cap n2v22_1m --nq 1048576
cap dw16 --app deepwalk --scale 16
cap dw22_1m --app deepwalk --scale 22 --nq 1048576
cap mp24_2m --app metapath --scale 24 --nq 2097152
cap ppr24_hub_256k --app ppr --scale 24 --queries hub --nq 262144
cap n2v22_lognormal_1m --weights lognormal --nq 1048576
ls -la $O | head -30
