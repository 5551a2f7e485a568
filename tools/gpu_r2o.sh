#!/bin/bash
# Round 2 o: ncu --set full of the fused build's TN dU (layer 1), NT update (layer 1) and the fused head.
O=gpurun_out/r2o
mkdir -p $O
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_f16x3 -s 2 -c 1 -o $O/tn_du1 $B > $O/ncu_tn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3_kernel -s 3 -c 1 -o $O/nt_upd1 $B > $O/ncu_nt.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3_kernel -s 5 -c 1 -o $O/nt_head $B > $O/ncu_head.log 2>&1
