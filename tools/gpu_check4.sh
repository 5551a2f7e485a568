#!/bin/bash
O=gpurun_out
./tools/probes/overlap_probe > $O/overlap_probe.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
