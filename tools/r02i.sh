make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py -m gpu -x -q > gpurun_out/r02i_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r02i_gputest.log
bash tools/ab_pairs.sh r02i "base::"
