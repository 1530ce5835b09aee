mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_suite.py -m gpu -q -rA -k "compat or reference_suite or switches" > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|PASSED|FAILED|xfail|Error|error" gpurun_out/pytest_gpu8.log | tail -40
