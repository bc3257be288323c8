# k_near_leaves: float-sqrt decisions with exact fallback; shard-share projection of the full-size legs
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r04k_gputest.log 2>&1; echo gputest rc=$?; tail -3 gpurun_out/r04k_gputest.log
bash tools/ab_pairs.sh r04k "head::" 2>&1 | grep -E "^==|pair_stage_ms|k_near_leaves|k_self|k_near_c8"
python tools/shard_share.py gpurun_out/r04k_shard_share.json > gpurun_out/r04k_shard_share.log 2>&1; tail -3 gpurun_out/r04k_shard_share.log | cut -c1-1200
