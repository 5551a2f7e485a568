#!/bin/bash
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 1200 python bench.py --config rmat --no-cpu-baseline --steps 3 > $O/bench_rmat.json 2> $O/bench_rmat.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $O/bench_rmat.err
timeout 1200 python bench.py --config rmat --scale 0.5 --no-cpu-baseline --steps 3 > $O/bench_rmat05.json 2> $O/bench_rmat05.err
