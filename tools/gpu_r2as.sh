#!/bin/bash
# Round 2 as: mid rows with narrow H as two 16-lane rows per warp — bitwise tests, Reddit / products A/B.
O=gpurun_out/r2as
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_fused_top.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
run() {  # label, cfg, env...
  env "${@:3}" timeout 600 python bench.py --config $2 --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1 $2', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if k.startswith('spmm')}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run new reddit
  run old reddit SC_LIB=variants/base/libsagecut_cuda.so
  run new products
  run old products SC_LIB=variants/base/libsagecut_cuda.so
done
