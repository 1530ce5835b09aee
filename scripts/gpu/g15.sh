mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_distributed.py -q -x > gpurun_out/pytest15.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest15.log
