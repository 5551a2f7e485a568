#!/bin/bash
# A/B kernel timing under ncu (launch durations + SM clock), alternating library builds:
#   tools/ab_kernels.sh "WORKLOAD ARGS" KERNEL_REGEX LIB1 LIB2 ... ("-" = in-tree build)
W=$1; K=$2; shift 2
for rep in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = "-" ]; then unset SC_LIB; else export SC_LIB=$lib; fi
    timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:$K -c 1 python tools/profile_kernels.py $W 2>&1 \
      | grep -E "duration|per_second|bytes" | awk -v l="$lib" '{printf "%s=%s%s ", $1, $3, $2} END {print " <- " l}' \
      | sed -e 's/gpu__time_duration.sum/t/' -e 's/sm__cycles_elapsed.avg.per_second/clk/' -e 's/dram__bytes_read.sum/rd/' -e 's/dram__bytes_write.sum/wr/'
  done
done
