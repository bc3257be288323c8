# grouped k_self (GS = 16 default): GPU parity, then A/B of GS / nodes / samples
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r03c_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r03c_gputest.log
bash tools/ab_pairs.sh r03c "gs16::" "gs32:build/variants/gs32/libvp_b200.so" "gs16n1:build/variants/gs16n1/libvp_b200.so" "gs16s6:build/variants/gs16s6/libvp_b200.so"
