#!/bin/bash
# Round 2 ae: narrow aggregation occupancy (min resident blocks 1 = none, 4, 5, 6).
O=gpurun_out/r2ae
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_spmm.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k.startswith('spmm')}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run mb1 SC_LIB=variants/nb1/libsagecut_cuda.so
  run mb4
  run mb5 SC_LIB=variants/nb5/libsagecut_cuda.so
  run mb6 SC_LIB=variants/nb6/libsagecut_cuda.so
done
