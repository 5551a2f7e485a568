#!/bin/bash
# Round 2 s: Xp products with the wide operand on the TN kernel's M side — tests + bench.
O=gpurun_out/r2s
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fused_top.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('swap', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>0.5}, d['loss_first_last'])" >> $O/ab.txt
done
