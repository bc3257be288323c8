make -j8 all > gpurun_out/r02d_build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/r02d_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02d_gputest.log 2>&1; echo gputest rc=$?
tail -5 gpurun_out/r02d_gputest.log
python bench.py --mode pairs --steps 3 --warmup 1 > gpurun_out/r02d_pairs.log 2>&1; echo pairs rc=$?
tail -c 1500 gpurun_out/r02d_pairs.log
bash tools/prof_kernels.sh r02d --mode pairs --steps 1 --warmup 1 -- k_self k_near_c8 k_psum_tgt k_near_int k_lists k_near_leaves
ls -la gpurun_out/
