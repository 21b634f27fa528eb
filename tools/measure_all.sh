#!/bin/bash
# Bench every config once (1 GPU) + the cfg3 launch list and ncu captures of
# the IVF kernels.  Outputs under gpurun_out/ (copy summaries to profiles/).
R=${ROUND:-r01}
for c in cfg1 cfg0 cfg2 cfg4 cfg3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.log 2>&1
done
timeout 900 bash tools/launchlist.sh gpurun_out/${R}_launches_cfg3.csv --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline
for k in ivf_list_kernel probe_select ivf_theta; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 \
    -o gpurun_out/${R}_${k}_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_ncu_$k.log 2>&1
done
echo measure done
