#!/bin/bash
O=gpurun_out
rm -f $O/diag.txt
for gm in auto simt; do timeout 600 python tools/diag_grads.py 47 $gm 20000 200000 >> $O/diag.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "staged or hubs" > $O/pytest_sel.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
