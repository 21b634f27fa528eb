for c in cfg1 cfg0 cfg2; do for sd in 8 16 64 128; do
BENCH_ARGS="--sample-div $sd" R=r02sw_${sd} CFGS="$c" bash tools/r02_step.sh | sed "s/^/sd=$sd /"
done; done
