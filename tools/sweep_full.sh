#!/bin/bash
# bench.py (config 2) + full-size configs $FULLCFG (default 5; FMM) per built variant under build/variants/*/libvp_b200.so
for d in build/variants/*/; do
  n=$(basename $d)
  VP_B200_LIB=$d/libvp_b200.so python bench.py --no-cpu-baseline --steps 5 > gpurun_out/sweep_$n.log 2>&1
  tail -1 gpurun_out/sweep_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['split_ms']; print('$n', round(d['value']), round(s['far'],2), round(s['near'],2), round(s['self'],3), round(d['alt_far_method']['ms_per_step'],3))" || tail -3 gpurun_out/sweep_$n.log
  for cfg in ${FULLCFG:-5}; do
    VP_B200_LIB=$d/libvp_b200.so python tools/full_config.py --config $cfg --check ${CHECK:-0} > gpurun_out/sweepfull_$n.log 2>&1
    tail -1 gpurun_out/sweepfull_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('   config$cfg', {k: round(v, 2) for k, v in d['device_ms'].items()}, d['u_rel_err_vs_oracle'])" || tail -3 gpurun_out/sweepfull_$n.log
  done
done
