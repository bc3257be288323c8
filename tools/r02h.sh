make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
bash tools/prof_kernels.sh r02h --mode pairs --steps 1 --warmup 1 -- k_self k_near_c8 k_psum_tgt k_near_int
