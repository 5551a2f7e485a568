#!/bin/bash
O=gpurun_out
rm -f $O/ab4.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
for rep in 1 2; do
for lib in variants/base2/libsagecut_cuda.so -; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib; fi
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab4.txt
done; done
