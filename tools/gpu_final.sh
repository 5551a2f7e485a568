#!/bin/bash
# Round-end evidence: full GPU suite, smoke, bench (+ reference arm), launch list, ncu captures.
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 6 -c 2 -o $O/spmm_full -f $B > $O/ncu_spmm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 1 -c 2 -o $O/tn_full -f $B > $O/ncu_tn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3_kernel -s 2 -c 2 -o $O/nt_full -f $B > $O/ncu_nt.log 2>&1
