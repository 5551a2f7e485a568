#!/bin/bash
# Round 2 m: L2 prefetch ahead of the GEMM loaders (TN distance, NT next tile) A/B; emulation / feature-row tests.
O=gpurun_out/r2m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x -k "emulated or feature_rows" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
}
for rep in 1 2; do
  run base
  run tnpf4 SC_TN_PF=4
  run tnpf8 SC_TN_PF=8
  run tnpf16 SC_TN_PF=16
  run ntpf SC_NT_PF=1
  run both8 SC_TN_PF=8 SC_NT_PF=1
done
