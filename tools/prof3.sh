#!/bin/bash
# usage (on the GPU box): tools/prof3.sh <tag> "<demangled-name regex>:<skip>:<count>" ...
# like prof2.sh but matches the demangled kernel name (template arguments
# included, e.g. "k_far<" without matching k_far_reduce).
set -e
TAG=$1; shift
CMD=${PROF_CMD:-"python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fmm"}
i=0
for SPEC in "$@"; do
  K=${SPEC%%:*}; R=${SPEC#*:}; S=${R%%:*}; C=${R#*:}
  REP=/tmp/${TAG}_$i
  ncu -f --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$K" -s $S -c $C \
      -o $REP $CMD > gpurun_out/${TAG}_ncu_$i.log 2>&1 || true
  if [ -f $REP.ncu-rep ]; then
    python tools/ncu_summary.py $REP.ncu-rep > gpurun_out/${TAG}_summary_$i.txt 2>&1 || true
    ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_$i.csv 2>/dev/null || true
    ncu -i $REP.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass_$i.csv 2>/dev/null || true
  fi
  i=$((i+1))
done
