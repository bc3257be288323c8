make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "far or shard or u_config" > gpurun_out/r02u_gputest.log 2>&1; echo gputest rc=$?; tail -1 gpurun_out/r02u_gputest.log
for tpt in auto 8 4; do
  if [ $tpt = auto ]; then unset VP_FAR_TPT; else export VP_FAR_TPT=$tpt; fi
  python bench.py --stride 2048 --steps 5 --warmup 3 --no-pairs --no-fmm --no-cpu-baseline > gpurun_out/r02u_s2048_$tpt.log 2>&1
  echo "stride 2048 tpt=$tpt: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r02u_s2048_$tpt.log | head -1)"
done
unset VP_FAR_TPT
python bench.py --steps 3 --warmup 3 --no-pairs --no-fmm --no-cpu-baseline > gpurun_out/r02u_s256.log 2>&1
echo "stride 256 auto: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/r02u_s256.log | head -1)"
