for ct in 16384 8192 4096 32768 16384; do
BENCH_ARGS="--tc-chunk-tiles $ct --steps 3 --warmup 1" R=r02ck_$ct CFGS="cfg4" bash tools/r02_step.sh | sed "s/^/chunk=$ct /"
done
