#!/bin/bash
O=gpurun_out
rm -f $O/ab6.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest_parity.log 2>&1; echo "rc=$?" >> $O/pytest_parity.log
for rep in 1 2; do
for lib in variants/base3 variants/spmm_g32 variants/flat_g64 variants/flat_g128 - variants/pipe_g32 variants/pipe_g64; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib/libsagecut_cuda.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if 'spmm' in k})" >> $O/ab6.txt
done; done
