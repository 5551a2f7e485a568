#!/bin/bash
# Round 2 y: papers 128-float rows 4 vs 8 rows per warp (papers at 10 % scale, p = 128); scale parity refresh.
O=gpurun_out/r2y
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_spmm.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
SC_SPMM_NARROW128=8 timeout 900 python -m pytest tests/test_gpu_spmm.py -q -x > $O/pytest8.log 2>&1; echo "rc=$?" >> $O/pytest8.log
for rep in 1 2; do
  timeout 900 python bench.py --config papers --scale 0.1 --parts 128 --steps 3 --no-cpu-baseline 2>>$O/err.txt | tail -1 > $O/papers4_$rep.json
  SC_SPMM_NARROW128=8 timeout 900 python bench.py --config papers --scale 0.1 --parts 128 --steps 3 --no-cpu-baseline 2>>$O/err.txt | tail -1 > $O/papers8_$rep.json
done
SC_PARITY_OUT=$O/scale_parity_head.json timeout 1500 python -m pytest tests/test_gpu_scale_parity.py -q > $O/pytest_scale.log 2>&1; echo "rc=$?" >> $O/pytest_scale.log
timeout 1800 python tools/scale_parity.py --config products --steps 5 --out $O/scale_free_products_head.json > $O/scale_free.log 2>&1
