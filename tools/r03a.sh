# k_self line profile at HEAD (config 4 pair stage)
CMD="python bench.py --mode pairs --steps 1 --warmup 1"
ncu --set full --clock-control none --import-source on --kernel-name-base function -k k_self -s 1 -c 1 \
    -o gpurun_out/r03a_k_self $CMD > gpurun_out/r03a_ncu.log 2>&1 || true
ncu -i gpurun_out/r03a_k_self.ncu-rep --page source --csv --print-source sass > gpurun_out/r03a_k_self_sass.csv 2>/dev/null
ncu -i gpurun_out/r03a_k_self.ncu-rep --page raw --csv > gpurun_out/r03a_k_self_raw.csv 2>/dev/null
ls -la gpurun_out
