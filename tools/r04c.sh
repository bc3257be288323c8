# psum index diet, c8 ping-pong G registers (vs copy variant), list-build grid cell size
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04c_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r04c_gputest.log
bash tools/ab_pairs.sh r04c "head::" "c8copy:build/variants/c8copy/libvp_b200.so" "grid50::VP_GRID_SCALE=0.5" "grid25::VP_GRID_SCALE=0.25"
