# launch list and ncu summaries of the pair kernels at HEAD (symmetric rules)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/r05y_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py /tmp/r05y_launch.csv > gpurun_out/r05y_launches.txt; head -32 gpurun_out/r05y_launches.txt
bash tools/prof_kernels.sh r05y --mode pairs --steps 1 --warmup 1 -- k_self k_near_c8 k_psum_tgt k_near_cache_mma2 k_near_int k_lists
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_near_leaves$" -s 0 -c 1 \
    -f -o /tmp/r05y_leaves python bench.py --mode pairs --steps 1 --warmup 0 > /tmp/r05y_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r05y_leaves.ncu-rep > gpurun_out/r05y_ncu_k_near_leaves.txt 2>&1
rm -f gpurun_out/r05y_raw_*.csv gpurun_out/r05y_sass_*.csv
du -sh gpurun_out
