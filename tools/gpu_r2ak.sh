#!/bin/bash
# Round 2 ak: papers-shaped rank-0 share with the DBH partitioner (lower replication) vs random.
O=gpurun_out/r2ak
mkdir -p $O
timeout 2400 python bench.py --config papers --partitioner dbh --steps 3 --warmup 1 --no-cpu-baseline > $O/papers_dbh.json 2> $O/papers_dbh.err
timeout 900 python bench.py --config products --partitioner dbh --no-cpu-baseline > $O/products_dbh.json 2> $O/products_dbh.err
