#!/bin/bash
O=gpurun_out/r2
mkdir -p $O
rm -f $O/ab_e.txt
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -k "tn" > $O/pytest_gemm_e.log 2>&1; echo "rc=$?" >> $O/pytest_gemm_e.log
for sp in 0 1; do
  SC_LIB=variants/trace/libsagecut_cuda.so SC_TN_TRACE=1 SC_TN_SPLIT=$sp timeout 300 python tools/profile_kernels.py tn512 2446000 > $O/tn_trace_e_split$sp.txt 2>&1
done
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab_e.txt
}
for rep in 1 2; do
  run base SC_LIB=variants/base/libsagecut_cuda.so
  run dual SC_TN_DUAL=1 SC_TN_SPLIT=0
  run nodual SC_TN_DUAL=0 SC_TN_SPLIT=0
  run dual_split SC_TN_DUAL=1 SC_TN_SPLIT=1
done
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_all_e.log 2>&1; echo "rc=$?" >> $O/pytest_all_e.log
