#!/bin/bash
# Round 2 af: wide aggregation occupancy (min resident blocks none / 6 / 8).
O=gpurun_out/r2af
mkdir -p $O
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k.startswith('spmm')}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run base
  run wb6 SC_LIB=variants/wb6/libsagecut_cuda.so
  run wb8 SC_LIB=variants/wb8/libsagecut_cuda.so
done
