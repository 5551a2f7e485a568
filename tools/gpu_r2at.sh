#!/bin/bash
# Round 2 at: other configs at HEAD (reddit, er10k, rmat 1/4, rmat_full, papers random / NE).
O=gpurun_out/r2at
mkdir -p $O
timeout 900 python bench.py --config reddit --no-cpu-baseline > $O/bench_reddit.json 2> $O/bench_reddit.err
timeout 600 python bench.py --config er10k > $O/bench_er10k.json 2> $O/bench_er10k.err
timeout 900 python bench.py --config rmat --no-cpu-baseline > $O/bench_rmat.json 2> $O/bench_rmat.err
timeout 1800 python bench.py --config rmat_full --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_rmat_full.json 2> $O/bench_rmat_full.err
timeout 2400 python bench.py --config papers --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_papers.json 2> $O/bench_papers.err
timeout 900 python bench.py --partitioner ne --no-cpu-baseline > $O/bench_products_ne.json 2> $O/bench_products_ne.err
