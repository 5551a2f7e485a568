#!/bin/bash
# Round 2 t: evidence refresh at the composed + projected build: full GPU suite, smoke, headline bench
# (+ CPU baseline), reference arm, launch list, per-config aggregation DRAM traffic, other configs.
O=gpurun_out/r2t
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
python tools/ncu_traffic.py --config products > $O/traffic_products.log 2>&1
python tools/ncu_traffic.py --config reddit > $O/traffic_reddit.log 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
   python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 900 python bench.py --config reddit --no-cpu-baseline > $O/bench_reddit.json 2> $O/bench_reddit.err
timeout 1800 python bench.py --config rmat_full --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_rmat_full.json 2> $O/bench_rmat_full.err
