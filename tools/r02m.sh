make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02m_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r02m_gputest.log
bash tools/ab_pairs.sh r02m "base::"
tail -c 900 gpurun_out/r02m_base.log
