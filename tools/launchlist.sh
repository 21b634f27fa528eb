#!/bin/bash
# usage: tools/launchlist.sh OUT.csv [bench args...]  -- per-launch device times of
# this library's kernels inside bench.py's timed steps (NVTX range "timed";
# cold-cache, serialised: use for shares, not absolutes)
out=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" \
    -k 'regex:cand8|tables_u16|tables_p16|scan4|scan8|select|theta|qadc|tables_exact|bucket|build_b|build_bias|fill_u|gather|ivf|probe|utables|pair_|merge|dense_adc|cnorm|v_kernel' \
    --csv --log-file "$out" python bench.py "$@" > /dev/null 2>&1
