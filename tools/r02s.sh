make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
bash tools/ab_pairs.sh r02s "base::" "nodes4:build/variants/nodes4/libvp_b200.so:" "nodes1:build/variants/nodes1/libvp_b200.so:"
