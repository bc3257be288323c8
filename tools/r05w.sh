# final profile set of the round at HEAD (symmetric rules, k_self at 5 blocks/SM): tests, flop profile, bench lines, launch list, ncu summaries
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r05w_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r05w_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05w_smoke.log 2>&1; tail -1 gpurun_out/r05w_smoke.log
python tools/fp64_flops.py gpurun_out/r02_fp64_flops_config4.json > gpurun_out/r05w_fp64_flops.log 2>&1; echo flops rc=$?
cp gpurun_out/r02_fp64_flops_config4.json profiles/ 2>/dev/null
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r05w_bench.log 2>&1; echo bench rc=$?
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r05w_ref.log 2>&1; echo ref rc=$?
python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/r05w_bench2.log 2>&1; echo b2 rc=$?
tail -c 6000 gpurun_out/r05w_bench.log; tail -c 1500 gpurun_out/r05w_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/r05w_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py /tmp/r05w_launch.csv > gpurun_out/r05w_launches.txt; head -32 gpurun_out/r05w_launches.txt
bash tools/prof_kernels.sh r05w --mode pairs --steps 1 --warmup 1 -- k_self k_near_c8 k_psum_tgt k_near_cache_mma2 k_near_int k_lists
rm -f gpurun_out/r05w_raw_*.csv gpurun_out/r05w_sass_*.csv
du -sh gpurun_out
