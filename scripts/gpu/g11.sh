python -m pytest tests/test_gpu_fullsize.py -m gpu -q -rA > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|PASSED|passed|failed" gpurun_out/pytest_gpu11.log | tail -12
timeout 1500 python scripts/gpu/parity_sweep.py > gpurun_out/sweep11.jsonl 2> gpurun_out/sweep11.err; echo "sweep rc=$?"
cut -c1-120 gpurun_out/sweep11.jsonl
