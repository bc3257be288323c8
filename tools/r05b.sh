# k_near_c8 lane-per-leaf tail pass for the 33rd node (vs the padded fifth slot)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r05b_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r05b_gputest.log
bash tools/ab_pairs.sh r05b "tail::" "notail::VP_C8_NO_TAIL=1" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_self|k_psum"
