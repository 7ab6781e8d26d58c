#!/bin/bash
# A/B two library builds across the first-order configs.
for args in "--app ppr --scale 24 --queries hub --nq 2097152" "--app deepwalk --scale 22" "--app deepwalk --scale 16" "--app metapath --scale 24"; do
  bash scripts/gpu_abn.sh "$args" "$@" 2>&1 | sed "s|^|[$args] |"
done
