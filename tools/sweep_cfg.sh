#!/bin/bash
# run a full-size config once per built variant: tools/sweep_cfg.sh CONFIG
CFG=${1:-4}
for d in build/variants/*/; do
  n=$(basename $d)
  VP_B200_LIB=$d/libvp_b200.so python tools/full_config.py --config $CFG --check 10 > gpurun_out/sweepc_$n.log 2>&1
  tail -1 gpurun_out/sweepc_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', d['device_ms'])" || tail -3 gpurun_out/sweepc_$n.log
done
