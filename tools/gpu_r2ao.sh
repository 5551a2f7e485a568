#!/bin/bash
# Round 2 ao: register-resident warp softmax-CE for 64 < C <= 256 — parity tests + papers 10 % A/B.
O=gpurun_out/r2ao
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
grep -q "rc=0" $O/pytest.log || exit 0
for rep in 1 2; do
  timeout 900 python bench.py --config papers --scale 0.1 --parts 128 --steps 3 --no-cpu-baseline 2>>$O/err.txt | tail -1 > $O/new_$rep.json
  SC_LIB=variants/base/libsagecut_cuda.so timeout 900 python bench.py --config papers --scale 0.1 --parts 128 --steps 3 --no-cpu-baseline 2>>$O/err.txt | tail -1 > $O/old_$rep.json
done
