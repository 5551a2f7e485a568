#!/bin/bash
# Round 2 h: spmm_bwd A/B (arena build vs the previous commit's build), per-config traffic (fixed
# fwd/bwd split), launch list, TN dual ncu, compact/dual tests, then the reference's full-scale
# products partition on the box's CPU.
O=gpurun_out/r2h
mkdir -p $O
run() {  # label, env...
  env "${@:2}" timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('$1', round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k: round(v['ms_per_step'],1) for k,v in d['kernels'].items() if v['ms_per_step']>1})" >> $O/ab.txt
}
for rep in 1 2; do
  run base SC_LIB=variants/base/libsagecut_cuda.so
  run arena
  run arena_compact SC_COMPACT_ACTS=1
done
timeout 600 python -m pytest tests/test_gpu_memory_modes.py -q > $O/pytest_modes.log 2>&1; echo "rc=$?" >> $O/pytest_modes.log
for c in products reddit; do timeout 600 python tools/ncu_traffic.py --config $c > $O/traffic_$c.txt 2>&1; done
timeout 900 python tools/ncu_traffic.py --config rmat > $O/traffic_rmat.txt 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1
SC_TN_DUAL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_f16x3 -s 1 -c 1 -o $O/tn_dual python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_f16x3 -s 1 -c 1 -o $O/tn_du python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tn2.log 2>&1
timeout 2700 python bench.py --cpu-full-partition > $O/cpu_full.json 2> $O/cpu_full.err
cp profiles/r02_reference_full_partition.json $O/ 2>/dev/null
