#!/bin/bash
# run bench.py once per built variant under build/variants/*/libvp_b200.so
for d in build/variants/*/; do
  n=$(basename $d)
  VP_B200_LIB=$d/libvp_b200.so python bench.py --no-cpu-baseline --steps 5 > gpurun_out/sweep_$n.log 2>&1
  tail -1 gpurun_out/sweep_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['split_ms']; print('$n', round(d['value']), round(s['far'],2), round(s['near'],2), round(s['self'],2))" || tail -3 gpurun_out/sweep_$n.log
done
