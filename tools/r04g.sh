# SM-level co-residency of the near chain and the self/point-sum stream: persistent partial grids
bash tools/ab_pairs.sh r04g "head::" "c8g1::VP_C8_BPSM=1" "c8g1s3::VP_C8_BPSM=1 VP_SELF_BPSM=3" "c8g2s3::VP_C8_BPSM=2 VP_SELF_BPSM=3" "ngb1:build/variants/ngb1/libvp_b200.so" "ngb1g1:build/variants/ngb1/libvp_b200.so:VP_C8_BPSM=1" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_self|k_psum"
