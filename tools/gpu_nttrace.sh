#!/bin/bash
O=gpurun_out
export SC_LIB=variants/nttrace/libsagecut_cuda.so SC_TN_TRACE=1
python tools/profile_kernels.py nt 2446000 > $O/nttrace.txt 2>&1
python tools/profile_kernels.py nt512 2446000 >> $O/nttrace.txt 2>&1
