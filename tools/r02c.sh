make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
bash tools/fp64_peak.sh > gpurun_out/r02c_peak.log 2>&1
python bench.py --steps 3 --warmup 3 --no-fmm --no-pairs > gpurun_out/r02c_bench.log 2>&1; echo bench rc=$?
tail -c 2500 gpurun_out/r02c_bench.log
bash tools/prof_pairs.sh r02c k_near_leaves k_near_c8 k_self k_psum_tgt k_near_int k_lists
python tools/far_profile.py gpurun_out/r02c_far_kernel_config4.json > gpurun_out/r02c_far.log 2>&1; echo far rc=$?
python tools/launch_summary.py gpurun_out/r02c_launches.csv > gpurun_out/r02c_launches.txt 2>&1
cat gpurun_out/r02c_launches.txt | head -30; cat gpurun_out/r02c_fp64_flops.log; tail -3 gpurun_out/r02c_far.log; cat gpurun_out/r02c_peak.log
