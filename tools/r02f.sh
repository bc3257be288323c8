make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
bash tools/ab_pairs.sh r02f "base::" "self5:build/variants/self5/libvp_b200.so:" "old:build/variants/old/libvp_b200.so:VP_PSUM_COPIES=1"
