#!/bin/bash
O=gpurun_out
timeout 1200 python bench.py --config rmat --no-cpu-baseline --steps 3 > $O/bench_rmat.json 2> $O/bench_rmat.err
timeout 900 python bench.py --config reddit --no-cpu-baseline > $O/bench_reddit.json 2> $O/bench_reddit.err
timeout 600 python bench.py --config er10k > $O/bench_er10k.json 2> $O/bench_er10k.err
