#!/bin/bash
# Round 2 g: arena / compact activations on the GPU suite; products bench; R-MAT full size (20M / 1B, p = 16);
# per-config DRAM traffic of the aggregation; ncu --set full of the TN dual and NT dgrad kernels.
O=gpurun_out/r2g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_memory_modes.py tests/test_gpu_parity.py -q -x > $O/pytest_a.log 2>&1; echo "rc=$?" >> $O/pytest_a.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_products.json 2> $O/bench_products.err
timeout 1500 python bench.py --config rmat_full --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_rmat_full.json 2> $O/bench_rmat_full.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $O/bench_rmat_full.err
for c in products reddit; do timeout 600 python tools/ncu_traffic.py --config $c > $O/traffic_$c.txt 2>&1; done
timeout 900 python tools/ncu_traffic.py --config rmat > $O/traffic_rmat.txt 2>&1
cp profiles/ncu_traffic.json $O/ncu_traffic.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tn_f16x3 -s 4 -c 1 -o $O/tn_dual python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_tn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f16x3_kernel -s 12 -c 2 -o $O/nt python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/ncu_nt.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_all.log 2>&1; echo "rc=$?" >> $O/pytest_all.log
