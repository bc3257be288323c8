# FMM order sweep (calibration of eps_fmm -> order) and finer list-build grids
python tools/fmm_tolerance.py gpurun_out/r04d_fmm_order_sweep.json > gpurun_out/r04d_fmm.log 2>&1; tail -4 gpurun_out/r04d_fmm.log
BENCH_ARGS="" bash tools/ab_pairs.sh r04d "head::" "grid12::VP_GRID_SCALE=0.125" "grid18::VP_GRID_SCALE=0.18"
grep -h "t_list\|list_build" gpurun_out/r04d_head.log | cut -c1-300 | head -3
