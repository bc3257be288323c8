# monomial density samples in k_self: GPU parity + pair-stage A/B
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r03b_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r03b_gputest.log
bash tools/ab_pairs.sh r03b "mono::"
