#!/bin/bash
# usage: tools/prof.sh <kernel-regex> <out-name> [bench args...]  (run on the GPU box)
# One ncu --set full capture of the first matching launch inside bench.py's
# timed steps (NVTX range "timed"; SKIP=n skips the first n matches), after the
# same command ran clean without ncu.
K=$1; OUT=$2; shift 2
python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/${OUT}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k "regex:$K" -s ${SKIP:-0} -c 1 -o gpurun_out/$OUT \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/${OUT}_ncu.log 2>&1
echo "prof exit $?"
