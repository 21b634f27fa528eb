#!/bin/bash
# End-of-round validation + measurement (one GPU): gpu tests, smoke, every
# config's bench line, launch lists (cfg1, cfg3) and ncu --set full captures
# of the dominant kernels (cfg1 tcgen05 filter, cfg3 list scan).
R=${ROUND:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/${R}_final_gputests.log 2>&1; echo "exit $?" >> gpurun_out/${R}_final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_final_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${R}_final_smoke.log
timeout 600 python bench.py > gpurun_out/${R}_final_bench_cfg1.log 2>&1
for c in cfg0 cfg2 cfg4 cfg3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_final_bench_$c.log 2>&1
done
timeout 600 bash tools/launchlist.sh gpurun_out/${R}_final_launches_cfg1.csv --steps 2 --warmup 1 --no-cpu-baseline
timeout 900 bash tools/launchlist.sh gpurun_out/${R}_final_launches_cfg3.csv --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:scan4tc' -s 3 -c 3 \
  -o gpurun_out/${R}_final_scan4tc_cfg1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_final_ncu_cfg1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:ivf_list_kernel' -s 1 -c 1 \
  -o gpurun_out/${R}_final_ivf_list_cfg3 python bench.py --config cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_final_ncu_cfg3.log 2>&1
echo final done
