#!/bin/bash
# One GPU session: parity tests, smoke, bench line, ncu launch list, ncu full capture of the aggregation
# and the dominant GEMM.  Outputs under gpurun_out/.
set -x
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 6 -c 1 -o $O/spmm_full -f \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_spmm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn -s 4 -c 1 -o $O/tn_full -f \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3 -s 6 -c 1 -o $O/nt_full -f \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_nt.log 2>&1
ls -la $O
