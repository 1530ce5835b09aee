mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -q -x -rA > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|PASSED|FAILED|Error" gpurun_out/pytest_gpu6.log | tail -80
