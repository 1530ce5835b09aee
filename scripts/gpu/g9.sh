set -x
python -m pytest tests -m gpu -x -q -rA > gpurun_out/pytest_gpu9.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu9.log
timeout 1500 python scripts/gpu/parity_sweep.py > gpurun_out/sweep9.jsonl 2> gpurun_out/sweep9.err; echo "sweep rc=$?"
cat gpurun_out/sweep9.jsonl | cut -c1-400
