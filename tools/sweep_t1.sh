R=r02tg_def CFGS="cfg0" bash tools/r02_step.sh | sed "s/^/target=default /"
for t in 2047 6000 8191; do
PQS_P16_TARGET=$t R=r02tg_$t CFGS="cfg0" bash tools/r02_step.sh | sed "s/^/target=$t /"
done
for t in 4095 2047 16383; do
PQS_P16_TARGET=$t R=r02tg2_$t CFGS="cfg2" bash tools/r02_step.sh | sed "s/^/target=$t /"
done
