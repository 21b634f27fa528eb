for pd in 4 8 16; do for sd in 2 4; do
PQS_PREFIX_DIV=$pd PQS_S0_DIV=$sd R=r02pf_${pd}_${sd} CFGS="cfg1" bash tools/r02_step.sh | sed "s/^/pdiv=$pd s0div=$sd /"
done; done
