make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_r02.py -m gpu -x -q > gpurun_out/r02l_gputest.log 2>&1; echo gputest rc=$?; tail -15 gpurun_out/r02l_gputest.log
python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02l_bench2.log 2>&1; echo b2 rc=$?; tail -c 2500 gpurun_out/r02l_bench2.log
python bench.py --mode pairs --steps 5 --warmup 1 > gpurun_out/r02l_pairs.log 2>&1; echo pairs rc=$?; tail -c 1500 gpurun_out/r02l_pairs.log
