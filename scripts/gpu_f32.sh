#!/bin/bash
bash scripts/gpu_abn.sh "" lib_edge.so lib_f32.so
FW_FAC32=0 bash scripts/gpu_abn.sh "" lib_f32.so
