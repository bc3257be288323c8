#!/bin/bash
# usage (GPU box): tools/prof_kernels.sh <tag> <bench args...> -- <kernel> [kernel ...]
# One `ncu --set full` capture per kernel (second launch) of a bench command;
# reports go to /tmp (too large for gpurun_out), their raw-page CSV and a text
# summary (tools/ncu_summary.py) to gpurun_out/.
TAG=$1; shift
ARGS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do ARGS+=("$1"); shift; done
shift
for K in "$@"; do
  ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^$K\$" -s 1 -c 1 \
      -f -o /tmp/${TAG}_$K python bench.py "${ARGS[@]}" > /tmp/${TAG}_ncu_$K.log 2>&1
  ncu -i /tmp/${TAG}_$K.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_$K.csv 2>/dev/null
  python tools/ncu_summary.py /tmp/${TAG}_$K.ncu-rep > gpurun_out/${TAG}_ncu_$K.txt 2>&1
  ncu -i /tmp/${TAG}_$K.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_src_$K.csv 2>/dev/null
  python tools/sass_hot.py /tmp/${TAG}_src_$K.csv 40 gpurun_out/${TAG}_sass_$K.csv > gpurun_out/${TAG}_hot_$K.txt 2>&1
done
