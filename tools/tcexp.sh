#!/bin/bash
# quick tcgen05 Quick ADC timing: cfg1 bench line summary + a 20M-code cfg4-shaped shard
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
d=json.loads([x for x in open("gpurun_out/bench.log") if x.startswith("{")][-1])
print("cfg1 %.3e evals/s  %.4f ms/step  cands %.0f  scan %.4f ms  e2e %.3e" % (d["value"], d["ms_per_step"], d["candidates"]["mean_per_query"], d["roofline"]["kernel_ms"], d["e2e"]["value"]))
PY
for md in ${MODES:-0}; do
PQS_TC_MODE=$md timeout 300 python bench.py --config cfg4 --n-per-gpu 20000000 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/m$md.log 2>&1
MD=$md python - <<'PY'
import json, os
md=os.environ["MD"]
d=json.loads([x for x in open("gpurun_out/m%s.log" % md) if x.startswith("{")][-1])
print("cfg4-20M mode %s: scan %.2f ms frac %.3f value %.3e" % (md, d["roofline"]["kernel_ms"], d["roofline"]["frac"], d["value"]))
PY
done
