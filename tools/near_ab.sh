#!/bin/bash
# A/B of the cached-leaf kernels on full-size configs (FMM far field):
# default (k_near_c8) vs VP_NEAR_CG=1 (k_near_cg); device ms per stage.
for cfg in ${CONFIGS:-2 3 4 5}; do
  for v in c8 cg; do
    if [ $v = cg ]; then export VP_NEAR_CG=1; else unset VP_NEAR_CG; fi
    python tools/full_config.py --config $cfg --check 0 > gpurun_out/nab_${cfg}_$v.log 2>&1
    tail -1 gpurun_out/nab_${cfg}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config $cfg $v', round(d['device_ms']['t_near_ms'],2), round(d['device_ms']['t_total_ms'],2), d['leaves'], d['targets'])"
  done
done
unset VP_NEAR_CG
