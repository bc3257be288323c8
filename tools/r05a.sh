# symmetric 33-point rule (order 12) and 12/25-point rules (orders 6, 10): GPU parity and first numbers
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r05a_gputest.log 2>&1; echo gputest rc=$?; tail -5 gpurun_out/r05a_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r05a_smoke.log 2>&1; tail -1 gpurun_out/r05a_smoke.log
python bench.py --steps 5 --warmup 3 > gpurun_out/r05a_bench.log 2>&1; echo bench rc=$?; tail -c 6500 gpurun_out/r05a_bench.log
bash tools/ab_pairs.sh r05a "head::" 2>&1 | head -16
