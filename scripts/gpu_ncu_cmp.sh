#!/bin/bash
# Source-attributed ncu capture of the Node2Vec walk kernel under env settings.
# usage: gpu_ncu_cmp.sh "ENV=a" "ENV=b" ...   (NQ queries, default 262144)
NQ=${NQ:-262144}; O=gpurun_out/ncmp; mkdir -p $O
i=0
for ev in "$@"; do
  env $ev timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 \
    -o $O/p$i python bench.py --steps 1 --warmup 0 --nq $NQ --no-cpu-baseline --no-e2e $EXTRA > $O/run$i.log 2>&1
  echo "$ev ncu rc=$?"
  ncu -i $O/p$i.ncu-rep --page source --csv --print-source cuda,sass > $O/src$i.csv 2>/dev/null
  ncu -i $O/p$i.ncu-rep --page raw --csv > $O/raw$i.csv 2>/dev/null
  python scripts/ncu_lines.py $O/src$i.csv 25 > $O/lines$i.txt 2>&1; head -30 $O/lines$i.txt
  i=$((i+1))
done
