#!/bin/bash
# Round 2 i: tcgen05 issue-rate probe (SS / TS, N = 256 / 128 / 64); spmm_bwd placement A/B
# (arena vs padded arena vs separate dh2 vs compact vs the round's first build).
O=gpurun_out/r2i
mkdir -p $O
timeout 120 tools/probes/mma_rate > $O/mma_rate.txt 2>&1; echo "rc=$?" >> $O/mma_rate.txt
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
}
for rep in 1 2; do
  run base SC_LIB=variants/base/libsagecut_cuda.so SC_TN_DUAL=0
  run arena
  run pad SC_LIB=variants/pad/libsagecut_cuda.so
  run noalias SC_LIB=variants/noalias/libsagecut_cuda.so
  run compact SC_COMPACT_ACTS=1
done
