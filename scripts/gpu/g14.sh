mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "determin" > gpurun_out/pytest14.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest14.log
