# HEAD validation after container restore: GPU tests, smoke, default bench, pair-stage profile refresh
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04a_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r04a_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r04a_smoke.log 2>&1; tail -1 gpurun_out/r04a_smoke.log
python bench.py > gpurun_out/r04a_bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/r04a_bench.log | cut -c1-600
bash tools/prof_pairs.sh r04a k_self k_near_c8 k_psum_tgt
python tools/launch_summary.py gpurun_out/r04a_launches.csv | head -20
for K in k_self k_near_c8 k_psum_tgt; do python tools/ncu_summary.py gpurun_out/r04a_$K.ncu-rep > gpurun_out/r04a_ncu_$K.txt 2>&1; done
