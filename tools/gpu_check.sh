#!/bin/bash
# Quick GPU session: full gpu test suite, smoke, bench, partitioner timing.
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err
timeout 900 python tools/time_partitioners.py > $O/partitioners.json 2> $O/partitioners.err
