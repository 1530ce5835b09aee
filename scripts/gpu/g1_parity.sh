mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python scripts/parity_report.py needle c1 c2 c3 c4 > gpurun_out/parity1.jsonl 2> gpurun_out/parity1.err; echo "parity rc=$?"
cut -c1-3000 gpurun_out/parity1.jsonl
