#!/bin/bash
# Round 2 am: the reference's default partitioner (NE, partition.cpp:116-201) on products and papers.
O=gpurun_out/r2am
mkdir -p $O
timeout 900 python bench.py --partitioner ne --no-cpu-baseline > $O/products_ne.json 2> $O/products_ne.err
timeout 3000 python bench.py --config papers --partitioner ne --steps 3 --warmup 1 --no-cpu-baseline > $O/papers_ne.json 2> $O/papers_ne.err
