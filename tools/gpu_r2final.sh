#!/bin/bash
# Round 2 final: evidence at the final round-2 build — full GPU suite, smoke, aggregation DRAM traffic per config, headline bench
# (+ CPU baseline) x2, reference arm, launch list, ncu --set full of the aggregation (wide + narrow)
# and the TN / NT GEMMs, other configs (reddit, er10k, rmat 1/4, rmat_full, papers).
O=gpurun_out/r2final
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python tools/ncu_traffic.py --config products > $O/traffic_products.log 2>&1
python tools/ncu_traffic.py --config reddit > $O/traffic_reddit.log 2>&1
python tools/ncu_traffic.py --config rmat > $O/traffic_rmat.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench2.json 2> $O/bench2.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_kernel -s 2 -c 2 -o $O/spmm_wide -f $B > $O/ncu_spmm.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm_narrow -s 0 -c 2 -o $O/spmm_narrow -f $B > $O/ncu_narrow.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_f16x3_kernel -s 8 -c 1 -o $O/tn_du1 -f $B > $O/ncu_tn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3_kernel -s 3 -c 1 -o $O/nt_upd1 -f $B > $O/ncu_nt.log 2>&1
timeout 900 python bench.py --config reddit --no-cpu-baseline > $O/bench_reddit.json 2> $O/bench_reddit.err
timeout 600 python bench.py --config er10k > $O/bench_er10k.json 2> $O/bench_er10k.err
timeout 900 python bench.py --config rmat --no-cpu-baseline > $O/bench_rmat.json 2> $O/bench_rmat.err
timeout 1800 python bench.py --config rmat_full --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_rmat_full.json 2> $O/bench_rmat_full.err
timeout 2400 python bench.py --config papers --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_papers.json 2> $O/bench_papers.err
