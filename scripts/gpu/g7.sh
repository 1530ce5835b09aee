mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -rA --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|PASSED|FAILED|Error|error" gpurun_out/pytest_gpu7.log | tail -40
