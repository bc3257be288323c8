make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
bash tools/prof_kernels.sh r02g --mode pairs --steps 1 --warmup 1 -- k_self k_near_c8
cat gpurun_out/r02g_cudahot_k_self.txt | head -80
