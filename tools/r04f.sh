# k_near_c8 occupancy variants (warps per block x min blocks)
bash tools/ab_pairs.sh r04f "ng10:build/variants/ng10/libvp_b200.so" "ng12:build/variants/ng12/libvp_b200.so" "ngb3:build/variants/ngb3/libvp_b200.so" "ng6b3:build/variants/ng6b3/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_near_cg"
