#!/bin/bash
# Round 2 x: narrow aggregation limited to rows of <= 64 slots (+ warp-per-row pass) — tests, products, R-MAT.
O=gpurun_out/r2x
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_fused_top.py tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 > $O/products_$rep.json
  timeout 900 python bench.py --config rmat --no-cpu-baseline --steps 5 2>>$O/ab_err.txt | tail -1 > $O/rmat_$rep.json
done
