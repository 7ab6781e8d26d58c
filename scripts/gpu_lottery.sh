#!/bin/bash
# A/B/n of semantically equivalent builds on the default bench, 2 rounds
bash scripts/gpu_abn.sh "" "$@"
