# k_near_c8<5> (33-node rule) at 10 and 12 warps per block
bash tools/ab_pairs.sh r05d "ng10:build/variants/ng10/libvp_b200.so" "ng12:build/variants/ng12/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8"
