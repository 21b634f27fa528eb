R=r02th_def CFGS="cfg3" TESTS="tests/test_gpu_ivf_scale.py tests/test_gpu_parity.py tests/test_gpu_sharded_2rank.py" bash tools/r02_step.sh | sed "s/^/default /"
for cfgp in "4 2048" "6 1024" "8 768" "12 1024" "8 512"; do set -- $cfgp
PQS_THETA_PROBES=$1 PQS_THETA_SPL=$2 R=r02th_$1_$2 CFGS="cfg3" bash tools/r02_step.sh | sed "s/^/probes=$1 spl=$2 /"
done
