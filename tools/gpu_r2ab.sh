#!/bin/bash
# Round 2 ab: toggles at the current build: dual TN launch, NT A'-in-TMEM off (the 48-wide P / Q GEMMs), TN stagger off.
O=gpurun_out/r2ab
mkdir -p $O
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run base
  run dual SC_TN_DUAL=1
  run nttm0 SC_NT_TM=0
  run nostag SC_TN_STAGGER=0
done
