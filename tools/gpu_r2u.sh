#!/bin/bash
# Round 2 u: narrow aggregation as LPR x CPL lanes, inv-scaled sums fused (no scale_rows) — tests + A/B.
O=gpurun_out/r2u
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_fused_top.py tests/test_gpu_multilabel.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('lprcpl', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>0.5}, d['roofline']['frac'], d['loss_first_last'])" >> $O/ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:spmm -c 12 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/spmm_launches.csv 2>&1
