#!/bin/bash
# Round 2 ap: 30 timed products epochs at the final build (training progress and steady timing).
O=gpurun_out/r2ap
mkdir -p $O
timeout 1200 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > $O/bench30.json 2> $O/bench30.err
