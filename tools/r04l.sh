# full-size configs 3/4/5 at HEAD (FMM far field, parity sample) and the main k_near_leaves launch
for spec in "3:0" "4:0" "5:10" "5:16" "5:24"; do
  c=${spec%%:*}; q=${spec#*:}
  name=config${c}; [ "$c" = 5 ] && name=config5q${q}
  python tools/full_config.py --config $c --q $q --check 400 --out gpurun_out/r02_${name}_full_fmm.json > gpurun_out/r04l_${name}.log 2>&1
  tail -1 gpurun_out/r04l_${name}.log | cut -c1-700
done
ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:"^k_near_leaves$" -s 0 -c 1 \
    -f -o /tmp/r04l_leaves python bench.py --mode pairs --steps 1 --warmup 0 > /tmp/r04l_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r04l_leaves.ncu-rep > gpurun_out/r04l_ncu_k_near_leaves.txt 2>&1
ncu -i /tmp/r04l_leaves.ncu-rep --page source --csv --print-source sass > /tmp/r04l_src.csv 2>/dev/null
python tools/sass_hot.py /tmp/r04l_src.csv 40 > gpurun_out/r04l_hot_k_near_leaves.txt 2>&1
head -12 gpurun_out/r04l_ncu_k_near_leaves.txt
