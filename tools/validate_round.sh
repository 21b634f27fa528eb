#!/bin/bash
# Full validation of the tree on one GPU box: gpu tests, smoke, default bench,
# launch list and one ncu --set full capture of the tcgen05 filter.
R=${ROUND:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/${R}_gputests.log 2>&1; echo "gpu tests exit $?" >> gpurun_out/${R}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/${R}_smoke.log
timeout 600 python bench.py > gpurun_out/${R}_bench_default.log 2>&1; echo "bench exit $?" >> gpurun_out/${R}_bench_default.log
timeout 600 bash tools/profile_round.sh
echo validate done
