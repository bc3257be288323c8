make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02r_gputest.log 2>&1; echo gputest rc=$?; tail -15 gpurun_out/r02r_gputest.log
bash tools/ab_pairs.sh r02r "base::"
