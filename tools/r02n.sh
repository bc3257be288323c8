make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
bash tools/prof_kernels.sh r02n --mode pairs --steps 1 --warmup 1 -- k_lists k_near_leaves k_near_cache_mma
