#!/bin/bash
# A/B of several variants (variants/NAME) against the in-tree build through bench.py (2 reps).
#   tools/gpu_ab_multi.sh NAME1 NAME2 ...
O=gpurun_out
rm -f $O/ab.txt
for rep in 1 2; do
for lib in - "$@"; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=variants/$lib/libsagecut_cuda.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
done; done
