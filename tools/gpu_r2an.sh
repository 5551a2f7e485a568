#!/bin/bash
# Round 2 an: TN epilogue warps converting half of each stage's B' (SC_TN_EPI_CONV=1) — tests + A/B.
O=gpurun_out/r2an
mkdir -p $O
SC_TN_EPI_CONV=1 timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "tn" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run base
  run epiconv SC_TN_EPI_CONV=1
done
