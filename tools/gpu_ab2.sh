#!/bin/bash
O=gpurun_out
rm -f $O/ab2.txt
timeout 900 python tools/e2e_probe.py 4 > $O/e2e_probe.txt 2>&1
for rep in 1 2; do
for lib in variants/base/libsagecut_cuda.so -; do
  if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib; fi
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$lib', round(d['ms_per_step'],1), round(d['e2e']['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab2.txt
done; done
unset SC_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 1 -c 2 -o $O/tn_du2 -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tn_du2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
