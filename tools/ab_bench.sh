#!/bin/bash
# A/B of whole training steps: alternate library builds ("-" = in-tree) through bench.py.
#   tools/ab_bench.sh "BENCH ARGS" LIB1 LIB2 ...
A=$1; shift
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib; fi
    timeout 600 python bench.py $A --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(round(d['ms_per_step'],1), {k:round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['clocks']['sm_mhz'], '<- $lib')"
  done
done
