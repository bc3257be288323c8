# k_near_c8s: consecutive targets per warp (leaf stream), prefetches across targets
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04h_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r04h_gputest.log
bash tools/ab_pairs.sh r04h "stream::" "gridstride::VP_C8_GRIDSTRIDE=1" "noelpf:build/variants/noelpf/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_self|k_psum"
