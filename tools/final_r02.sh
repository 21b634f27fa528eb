#!/bin/bash
# Round-2 final validation + measurement on one GPU box (outputs under gpurun_out/r02z_*):
# gpu tests, smoke, the default bench line (with cpu_baseline) and the reference arm,
# every other config's bench line, launch lists and ncu --set full captures of the
# dominant kernels (each after its plain command exited 0).
R=r02z
mkdir -p gpurun_out
timeout 1500 python tests/parity_full.py cfg0 cfg1 cfg2 cfg3 cfg4 --out gpurun_out/parity_full_${R}.json > gpurun_out/${R}_parity.log 2>&1; echo "exit $?" >> gpurun_out/${R}_parity.log
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/${R}_gputests.log 2>&1; echo "exit $?" >> gpurun_out/${R}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${R}_smoke.log
timeout 900 python bench.py > gpurun_out/${R}_bench_default.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_reference.log 2>&1
for c in cfg1 cfg0 cfg2 cfg3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.log 2>&1
done
for c in cfg4 cfg1 cfg0 cfg2 cfg3; do
  timeout 600 bash tools/launchlist.sh gpurun_out/${R}_launches_$c.csv --config $c --steps 1 --warmup 1 --no-cpu-baseline
done
SKIP=5 timeout 600 bash tools/prof.sh scan4tc_kernel ${R}_scan4tc_cfg4 --config cfg4   # a main-range launch (the first is the prefix)
SKIP=1 timeout 600 bash tools/prof.sh scan8p ${R}_scan8p_cfg0 --config cfg0   # the second filter launch (7/8 of the tiles)
SKIP=1 timeout 600 bash tools/prof.sh scan8p ${R}_scan8p_cfg2 --config cfg2
timeout 600 bash tools/prof.sh ivf_list8 ${R}_list8_cfg3 --config cfg3
tail -n 3 gpurun_out/${R}_gputests.log gpurun_out/${R}_smoke.log
for f in gpurun_out/${R}_bench_*.log; do echo $f; tail -n 1 $f | cut -c1-400; done
