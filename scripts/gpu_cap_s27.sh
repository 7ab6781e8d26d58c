#!/bin/bash
O=gpurun_out/caps; mkdir -p $O
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o $O/n2v27_2m \
  python bench.py --scale 27 --nq 2097152 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/n2v27_2m.json 2> $O/n2v27_2m.err
echo "ncu rc=$?"
