#!/bin/bash
O=gpurun_out
for C in 47 61; do for gm in auto simt; do timeout 300 python tools/diag_grads.py $C $gm >> $O/diag.txt 2>&1; done; done
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
