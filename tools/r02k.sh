make -j8 all > /dev/null 2>&1 || echo BUILD FAILED
BENCH_ARGS="--near-cache-gb 40" bash tools/ab_pairs.sh r02k "d3_40gb::"
BENCH_ARGS="--near-cache-depth 1" bash tools/ab_pairs.sh r02k "d1::"
