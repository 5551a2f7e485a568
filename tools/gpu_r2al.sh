#!/bin/bash
# Round 2 al: NT operand stages / fp32 staging slots 4/4 (base) vs 3/5 vs 3/6.
O=gpurun_out/r2al
mkdir -p $O
for v in nt35 nt36; do
  SC_LIB=variants/$v/libsagecut_cuda.so timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "f16x3_matches" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
done
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run base
  run nt35 SC_LIB=variants/nt35/libsagecut_cuda.so
  run nt36 SC_LIB=variants/nt36/libsagecut_cuda.so
done
