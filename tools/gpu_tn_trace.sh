#!/bin/bash
O=gpurun_out
rm -f $O/tntrace3.txt
for v in tntrace tnnored tnnotr; do
  echo "== $v" >> $O/tntrace3.txt
  SC_LIB=variants/$v/libsagecut_cuda.so SC_TN_TRACE=1 python tools/profile_kernels.py tn512 2446000 2>&1 | grep -v wall | tail -1 >> $O/tntrace3.txt
done
