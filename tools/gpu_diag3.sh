#!/bin/bash
O=gpurun_out
rm -f $O/diag3.txt
for de in 1 0; do timeout 600 python tools/diag_part.py $de simt >> $O/diag3.txt 2>&1; done
