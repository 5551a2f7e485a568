#!/bin/bash
# Round 2 aj: TMA drain stores / reduce-adds with the L2 evict_last hint — bitwise test, A/B, DRAM bytes.
O=gpurun_out/r2aj
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -k "tn" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items() if v['ms_per_step']>1}, d['loss_first_last'])" >> $O/ab.txt
}
for rep in 1 2; do
  run hint
  run nohint SC_LIB=variants/base/libsagecut_cuda.so
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tn_f16x3_kernel -s 10 -c 1 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/tn_hint.csv 2>&1
