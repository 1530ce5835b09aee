mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest20.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest20.log
for c in c4 c1 c3; do CFG=$c bash scripts/gpu/ab_env.sh "BSR_X=0" "BSR_X=1"; done
