# HEAD check after returning k_near_c8 to 8 warps per block: GPU tests, pair stage, FMM evaluation
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r05f_gputest.log 2>&1; echo gputest rc=$?; tail -2 gpurun_out/r05f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/ab_pairs.sh r05f "head::" 2>&1 | grep -E "^==|pair_stage_ms|k_near_c8|k_self"
python tools/full_config.py --config 4 --check 200 2>&1 | tail -1 | cut -c1-700
