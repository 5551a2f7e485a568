#!/bin/bash
O=gpurun_out
rm -f $O/ab5.txt
for rep in 1 2; do
for lib in - variants/spmm_q8/libsagecut_cuda.so variants/spmm_q2/libsagecut_cuda.so variants/spmm_g32/libsagecut_cuda.so; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if 'spmm' in k})" >> $O/ab5.txt
done; done
