nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
( time python bench.py --steps 3 --warmup 3 ) > gpurun_out/r02b_bench.log 2>&1; echo bench rc=$?
tail -c 6000 gpurun_out/r02b_bench.log
( time python bench.py --impl reference --steps 3 --warmup 1 ) > gpurun_out/r02b_ref.log 2>&1; echo ref rc=$?
tail -c 3000 gpurun_out/r02b_ref.log
nproc; lscpu | grep -i "model name"
