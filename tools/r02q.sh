make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
python tools/fp64_flops.py gpurun_out/r02_fp64_flops_config4.json > gpurun_out/r02q_fp64_flops.log 2>&1; echo flops rc=$?
python tools/far_profile.py gpurun_out/r02_far_kernel_config4.json > gpurun_out/r02q_far.log 2>&1; echo far rc=$?
rm -f gpurun_out/r02_far_kernel_config4.ncu-rep
mkdir -p profiles_tmp; cp gpurun_out/r02_fp64_flops_config4.json gpurun_out/r02_far_kernel_config4.json profiles/ 2>/dev/null
( time python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02q_bench.log 2>&1; echo bench rc=$?
( time python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r02q_ref.log 2>&1; echo ref rc=$?
tail -c 5000 gpurun_out/r02q_bench.log; tail -c 1500 gpurun_out/r02q_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/r02q_launch.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py /tmp/r02q_launch.csv > gpurun_out/r02q_launches.txt; head -30 gpurun_out/r02q_launches.txt
