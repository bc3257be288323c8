# FMM: tolerance -> order, active-box downward pass: GPU tests, shard timing, order timing
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04e_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r04e_gputest.log
run() { # name, env, args
  env $2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/r04e_$1.csv python tools/fmm_shard.py $3 > gpurun_out/r04e_$1.log 2>&1
  python tools/launch_summary.py /tmp/r04e_$1.csv > gpurun_out/r04e_$1_launches.txt 2>&1
  echo "== $1"; tail -1 gpurun_out/r04e_$1.log; grep -E "fmm|k_far" gpurun_out/r04e_$1_launches.txt | head -8
}
run c4_shard_masked "A=1" "--config 4 --targets shard"
run c4_shard_allboxes "VP_FMM_ALL_BOXES=1" "--config 4 --targets shard"
run c4_all "A=1" "--config 4 --targets all"
run c4_all_eps8 "A=1" "--config 4 --targets all --eps 1e-8"
run c3_all "A=1" "--config 3 --targets all"
run c3_all_eps8 "A=1" "--config 3 --targets all --eps 1e-8"
