#!/bin/bash
# Round profile capture (run on the GPU box, one GPU):
#   launch list of the default bench step, ncu --set full of the Quick ADC
#   kernels of one step (tcgen05 histogram + prefix/main filter launches).
set -e
R=${ROUND:-r01}
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_cfg1.csv \
    -k 'regex:scan4|select|theta|qadc|tables_exact|bucket|build_b|build_bias|fill_u' \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:scan4tc' -s 3 -c 3 \
    -o gpurun_out/${R}_scan4tc_cfg1 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${R}_ncu.log 2>&1
echo "profile done"
