#!/bin/bash
# A/B: TN tests, then the in-tree library against variants/$1 through bench.py (2 reps).
O=gpurun_out
BASE=${1:-base}
rm -f $O/ab.txt
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -s > $O/pytest_gemm.log 2>&1; echo "rc=$?" >> $O/pytest_gemm.log
if grep -q "rc=0" $O/pytest_gemm.log; then
for rep in 1 2; do
for lib in variants/$BASE -; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib/libsagecut_cuda.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
done; done
fi
