# full-size configs 3/4/5 (FMM far field, parity sample) and one GPU's share of an 8-way run, symmetric rules
for spec in "3:0" "4:0" "5:10" "5:16" "5:24"; do
  c=${spec%%:*}; q=${spec#*:}
  name=config${c}; [ "$c" = 5 ] && name=config5q${q}
  python tools/full_config.py --config $c --q $q --check 400 --out gpurun_out/r02_${name}_full_fmm.json > gpurun_out/r05x_${name}.log 2>&1
  tail -1 gpurun_out/r05x_${name}.log | cut -c1-400
done
python tools/shard_share.py gpurun_out/r02_shard_share_config4.json > gpurun_out/r05x_shard_share.log 2>&1; tail -2 gpurun_out/r05x_shard_share.log | cut -c1-300
