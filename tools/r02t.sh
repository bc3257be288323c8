make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02t_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r02t_gputest.log
bash tools/ab_pairs.sh r02t "base::"
python bench.py --steps 3 --warmup 3 --no-pairs --no-fmm --no-cpu-baseline > gpurun_out/r02t_head.log 2>&1; tail -c 800 gpurun_out/r02t_head.log
