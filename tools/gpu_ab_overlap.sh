#!/bin/bash
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for rep in 1 2; do
for ov in 0 1; do
  SC_OVERLAP=$ov timeout 600 python bench.py --no-cpu-baseline > $O/bench_ov$ov.json 2>/dev/null
  python -c "
import json; d=json.load(open('$O/bench_ov$ov.json'))
print('overlap=$ov', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
done; done
