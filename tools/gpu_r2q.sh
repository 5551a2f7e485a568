#!/bin/bash
# Round 2 q: projected top-layer aggregation (PTA) — tests, A/B, full suite.
O=gpurun_out/r2q
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused_top.py tests/test_gpu_gemm.py -q -x > $O/pytest_fused.log 2>&1; echo "rc=$?" >> $O/pytest_fused.log
grep -q "rc=0" $O/pytest_fused.log || exit 0
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>0.5}, d['loss_first_last'], d['eval']['train_val_test'])" >> $O/ab.txt
}
for rep in 1 2; do
  run pta
  run nopta SC_PTA=0
done
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
