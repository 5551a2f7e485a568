#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "many_classes or sbm200 or config0" > $O/pytest_sm.log 2>&1; echo "rc=$?" >> $O/pytest_sm.log
bash tools/gpu_ab_multi.sh base11
