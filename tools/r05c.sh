# k_self at 16-lane groups: nodes per lane and resident blocks
bash tools/ab_pairs.sh r05c "n1:build/variants/n1/libvp_b200.so" "n3:build/variants/n3/libvp_b200.so" "n4:build/variants/n4/libvp_b200.so" "mb5:build/variants/mb5/libvp_b200.so" "mb4:build/variants/mb4/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_self"
