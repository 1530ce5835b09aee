mkdir -p gpurun_out
timeout 1100 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest19.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest19.log
CFG=c4 bash scripts/gpu/ab_env.sh "BSR_X=0"
CFG=c1 bash scripts/gpu/ab_env.sh "BSR_X=0"
