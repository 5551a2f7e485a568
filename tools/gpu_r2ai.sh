#!/bin/bash
# Round 2 ai: ncu --set full of the final build's TN dU (layer 1) and NT update (layer 1).
O=gpurun_out/r2ai
mkdir -p $O
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_f16x3_kernel -s 10 -c 1 -o $O/tn_du1 -f $B > $O/ncu_tn.log 2>&1
