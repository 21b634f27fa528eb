#!/bin/bash
# One iteration on the GPU box: selected tests, then selected bench configs.
# usage: R=tag TESTS="tests/a.py tests/b.py" CFGS="cfg0 cfg2" bash tools/r02_step.sh
R=${R:-r02s}
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 2400 python -m pytest $TESTS -q -m gpu -x > gpurun_out/${R}_tests.log 2>&1; echo "exit $?" >> gpurun_out/${R}_tests.log
  tail -n 15 gpurun_out/${R}_tests.log
fi
for c in $CFGS; do
  timeout 900 python bench.py --config $c --no-cpu-baseline $BENCH_ARGS > gpurun_out/${R}_bench_$c.log 2>&1
  tail -n 1 gpurun_out/${R}_bench_$c.log | python -c "
import json,sys
for l in sys.stdin:
    try:
        j=json.loads(l); r=j['roofline']; print('$c', '%.3e'%j['value'], 'ms', round(j['ms_per_step'],3), 'kernel_ms', r.get('kernel_ms'), 'frac', round(r['frac'],3), 'cand', j.get('candidates',{}).get('mean_per_query'), j['clocks'])
    except Exception as e: print('$c', 'bad line', e, l[:300])
"
done
