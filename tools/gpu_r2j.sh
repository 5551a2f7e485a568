#!/bin/bash
# Round 2 j: A'-in-TMEM NT kernel (fp64 checks first), the aggregation with a compile-time ReLU-bits
# variant; products A/B: default vs SC_NT_TM=0 vs compact.
O=gpurun_out/r2j
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > $O/pytest_gemm.log 2>&1; echo "rc=$?" >> $O/pytest_gemm.log
grep -q "rc=0" $O/pytest_gemm.log || exit 0
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
}
for rep in 1 2; do
  run tm
  run notm SC_NT_TM=0
  run tm_compact SC_COMPACT_ACTS=1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_memory_modes.py tests/test_gpu_scale_parity.py -q -x > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_nt_tm -s 1 -c 2 -o $O/nt_tm python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_nt.log 2>&1
