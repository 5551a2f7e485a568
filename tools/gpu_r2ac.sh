#!/bin/bash
# Round 2 ac: narrow forward-add with the addend row / inv prefetched — bitwise test + A/B vs the previous build.
O=gpurun_out/r2ac
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_fused_top.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run new
  run old SC_LIB=variants/base/libsagecut_cuda.so
done
