#!/bin/bash
# Round 2 ad: compact activations (ReLU sign bits for every layer's transposed aggregation) vs default.
O=gpurun_out/r2ad
mkdir -p $O
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run default
  run compact SC_COMPACT_ACTS=1
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmm_kernel -c 8 --csv env SC_COMPACT_ACTS=1 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/spmm_compact.csv 2>&1
