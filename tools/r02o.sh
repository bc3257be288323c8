make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "near or list or u_config" > gpurun_out/r02o_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r02o_gputest.log
bash tools/ab_pairs.sh r02o "base::"
