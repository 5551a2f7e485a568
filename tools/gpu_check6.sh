#!/bin/bash
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "unaligned or sbm200 or config0" > $O/pytest_sel.log 2>&1; echo "rc=$?" >> $O/pytest_sel.log
timeout 900 python bench.py --config reddit --no-cpu-baseline > $O/bench_reddit.json 2> $O/bench_reddit.err
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
