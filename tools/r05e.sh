# k_near_c8<5> at 9 and 11 warps per block
bash tools/ab_pairs.sh r05e "ng9:build/variants/ng9/libvp_b200.so" "ng11:build/variants/ng11/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8"
