#!/bin/bash
# usage (on the GPU box): tools/prof2.sh <tag> "<kernel regex>:<skip>:<count>" ...
# plain run, launch list, then one `ncu --set full` capture per spec, reduced
# on the box to a metric summary + raw csv + source csv (reports are large).
set -e
TAG=$1; shift
CMD=${PROF_CMD:-"python bench.py --steps 1 --warmup 3 --no-cpu-baseline"}
$CMD > gpurun_out/${TAG}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > /dev/null 2>&1
i=0
for SPEC in "$@"; do
  K=${SPEC%%:*}; R=${SPEC#*:}; S=${R%%:*}; C=${R#*:}
  REP=/tmp/${TAG}_$i
  ncu -f --set full --clock-control none --import-source on --kernel-name-base function -k regex:$K -s $S -c $C \
      -o $REP $CMD > gpurun_out/${TAG}_ncu_$i.log 2>&1 || true
  if [ -f $REP.ncu-rep ]; then
    python tools/ncu_summary.py $REP.ncu-rep > gpurun_out/${TAG}_summary_$i.txt 2>&1 || true
    ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_$i.csv 2>/dev/null || true
    ncu -i $REP.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass_$i.csv 2>/dev/null || true
    if [ -n "$KEEP" ]; then cp $REP.ncu-rep gpurun_out/; fi
  fi
  i=$((i+1))
done
