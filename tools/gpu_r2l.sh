#!/bin/bash
# Round 2 l: sparse vertex cut (bit-exact tests), papers100M-shaped config (rank-0 emulation).
O=gpurun_out/r2l
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_facade.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --config papers --scale 0.05 --parts 128 --steps 2 --warmup 1 --no-cpu-baseline > $O/papers_s005.json 2> $O/papers_s005.err
timeout 2400 python bench.py --config papers --steps 3 --warmup 1 --no-cpu-baseline > $O/papers_full.json 2> $O/papers_full.err
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> $O/papers_full.err
