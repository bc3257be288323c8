make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_r02.py -m gpu -x -q -k "self or u_config or full_size or evaluate_device" > gpurun_out/r02e_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r02e_gputest.log
bash tools/ab_pairs.sh r02e "base::" "self5:build/variants/self5/libvp_b200.so:" "self4:build/variants/self4/libvp_b200.so:" "pc1::VP_PSUM_COPIES=1" "pc2::VP_PSUM_COPIES=2" "pc8::VP_PSUM_COPIES=8"
