#!/bin/bash
O=gpurun_out/r2
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_gemm.py -q > $O/pytest_gemm_b.log 2>&1; echo "rc=$?" >> $O/pytest_gemm_b.log
timeout 900 python -m pytest tests/test_gpu_multilabel.py tests/test_gpu_multirank.py tests/test_gpu_facade.py -q > $O/pytest_b.log 2>&1; echo "rc=$?" >> $O/pytest_b.log
rm -f $O/ab_b.txt
for rep in 1 2; do for lib in variants/base/libsagecut_cuda.so -; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab_b.txt
done; done
unset SC_LIB
SC_PARITY_OUT=$O/scale_parity.json timeout 1800 python -m pytest tests/test_gpu_scale_parity.py -q -s > $O/pytest_scale.log 2>&1; echo "rc=$?" >> $O/pytest_scale.log
timeout 1200 python tools/scale_parity.py --config products --steps 5 --out $O/scale_free_products.json > $O/scale_free.log 2>&1
