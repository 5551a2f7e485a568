#!/bin/bash
O=gpurun_out
rm -f $O/ab3.txt
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x -k "gemm or tn or sbm200 or er10k" > $O/pytest_gemm.log 2>&1; echo "rc=$?" >> $O/pytest_gemm.log
for rep in 1 2; do
for d in 0 1; do
  SC_TN_DIRECT=$d timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('direct=$d', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab3.txt
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 1 -c 2 -o $O/tn_du3 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tn_du3.log 2>&1
timeout 900 python tools/e2e_probe.py 4 > $O/e2e_probe.txt 2>&1
