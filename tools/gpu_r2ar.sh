#!/bin/bash
# Round 2 ar: softmax-CE row kernel occupancy (min blocks none / 8 / 12).
O=gpurun_out/r2ar
mkdir -p $O
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['kernels']['loss']['ms_per_step'],3), d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run base
  run sm8 SC_LIB=variants/sm8/libsagecut_cuda.so
  run sm12 SC_LIB=variants/sm12/libsagecut_cuda.so
done
