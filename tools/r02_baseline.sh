#!/bin/bash
# Re-validation of the restored tree on one GPU box: gpu tests, smoke, every config's bench line.
R=${ROUND:-r02v}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/${R}_gputests.log 2>&1; echo "exit $?" >> gpurun_out/${R}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "exit $?" >> gpurun_out/${R}_smoke.log
for c in cfg1 cfg0 cfg2 cfg3; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.log 2>&1
done
timeout 900 python bench.py > gpurun_out/${R}_bench_default.log 2>&1
tail -n 3 gpurun_out/${R}_gputests.log gpurun_out/${R}_smoke.log
tail -n 1 gpurun_out/${R}_bench_*.log
