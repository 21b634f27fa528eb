for c in cfg0 cfg2; do for sd in 32 48 64 96 128; do
BENCH_ARGS="--sample-div $sd" R=r02sw_${sd} CFGS="$c" bash tools/r02_step.sh | sed "s/^/sd=$sd /"
done; done
