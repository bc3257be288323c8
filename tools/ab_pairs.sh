#!/bin/bash
# A/B of library variants on the full-size pair stage (GPU box):
#   tools/ab_pairs.sh TAG "name:lib_path:ENV=VAL ..." ...
# per variant: bench.py --mode pairs (live pair-stage ms) and an ncu launch
# list of the pair kernels (isolated, serialised ms).
TAG=$1; shift
for V in "$@"; do
  NAME=${V%%:*}; REST=${V#*:}; LIB=${REST%%:*}; ENVS=${REST#*:}
  [ "$ENVS" = "$REST" ] && ENVS=""
  [ -n "$LIB" ] && export VP_B200_LIB=$LIB || unset VP_B200_LIB
  env $ENVS python bench.py --mode pairs --steps 3 --warmup 1 ${BENCH_ARGS} > gpurun_out/${TAG}_${NAME}.log 2>&1
  env $ENVS ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file /tmp/${TAG}_${NAME}.csv python bench.py --mode pairs --steps 1 --warmup 0 ${BENCH_ARGS} > /dev/null 2>&1
  python tools/launch_summary.py /tmp/${TAG}_${NAME}.csv > gpurun_out/${TAG}_${NAME}_launches.txt 2>&1
  echo "== $NAME ($LIB $ENVS)"; tail -1 gpurun_out/${TAG}_${NAME}.log | python -c "import json,sys; d=json.loads(sys.stdin.read())['pair_stage']; print('pair_stage_ms', round(d['pair_stage_ms'],2), 'step', round(d['ms_per_step'],2))"
  head -12 gpurun_out/${TAG}_${NAME}_launches.txt
done
unset VP_B200_LIB
