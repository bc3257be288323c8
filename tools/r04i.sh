# k_near_c8s grid-stride with look-ahead (vs k_near_c8), psum two-stage list heads at several occupancies
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04i_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r04i_gputest.log
bash tools/ab_pairs.sh r04i "c8s::" "c8::VP_C8_GRIDSTRIDE=1" "noelpf:build/variants/noelpf/libvp_b200.so" "psb4:build/variants/psb4/libvp_b200.so" "psb5:build/variants/psb5/libvp_b200.so" "psb6:build/variants/psb6/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_self|k_psum"
