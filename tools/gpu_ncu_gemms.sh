#!/bin/bash
# ncu --set full of the update GEMM (dual source, K=512), the dU weight gradient (N2=512) and dW (N2=256).
O=gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 1 -c 2 -o $O/tn_du -f $B > $O/ncu_tn_du.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3_kernel -s 3 -c 1 -o $O/nt_upd -f $B > $O/ncu_nt_upd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:softmax_ce -s 0 -c 1 -o $O/loss -f $B > $O/ncu_loss.log 2>&1
