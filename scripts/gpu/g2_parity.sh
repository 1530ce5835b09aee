mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu2.log
timeout 1500 python scripts/parity_report.py needle c3 c4 > gpurun_out/parity2.jsonl 2> gpurun_out/parity2.err; echo "parity rc=$?"
cat gpurun_out/parity2.jsonl; tail -5 gpurun_out/parity2.err
