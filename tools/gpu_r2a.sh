#!/bin/bash
# Round-2 session A: new parity tests (multi-label, multi-rank, headline-scale), bench, free-running scale parity.
O=gpurun_out/r2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multilabel.py tests/test_gpu_multirank.py -q > $O/pytest_a.log 2>&1; echo "rc=$?" >> $O/pytest_a.log
SC_PARITY_OUT=$O/scale_parity.json timeout 1800 python -m pytest tests/test_gpu_scale_parity.py -q -s > $O/pytest_scale.log 2>&1; echo "rc=$?" >> $O/pytest_scale.log
timeout 600 python bench.py > $O/bench_a.json 2> $O/bench_a.err
timeout 1200 python tools/scale_parity.py --config products --steps 5 --out $O/scale_free_products.json > $O/scale_free.log 2>&1
