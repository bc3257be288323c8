# k_self halvings + GS=8 variant, near-cache mma2 (V tile resident): GPU parity, A/B, k_self line profile
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04b_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r04b_gputest.log
bash tools/ab_pairs.sh r04b "head::" "mma1::VP_NEAR_CACHE_MMA1=1" "gs8:build/variants/gs8/libvp_b200.so"
PROF_CMD="python bench.py --mode pairs --steps 1 --warmup 1" bash tools/prof3.sh r04b "k_self<:1:1" "k_near_cache_mma2:1:1"
python tools/sass_hot.py gpurun_out/r04b_sass_0.csv 40 gpurun_out/r04b_k_self_inst.csv > gpurun_out/r04b_k_self_hot.txt 2>&1
python tools/sass_lines.py gpurun_out/r04b_k_self_inst.csv k_selfILi6ELi16 60 > gpurun_out/r04b_k_self_lines.txt 2>&1
rm -f gpurun_out/r04b_sass_*.csv gpurun_out/r04b_raw_*.csv
du -sh gpurun_out
