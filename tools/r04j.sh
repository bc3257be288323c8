# k_self L1 prefetch of the next item's inputs
bash tools/ab_pairs.sh r04j "selfpf::" "selfnopf:build/variants/selfnopf/libvp_b200.so" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_self|k_psum"
