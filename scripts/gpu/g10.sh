python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest rc=$?"
grep -E "FAILED|passed|failed" gpurun_out/pytest_gpu10.log | tail -5
CFG=c4 bash scripts/gpu/ab.sh cur nox cur nox
CFG=c1 bash scripts/gpu/ab.sh cur nox
timeout 1500 python scripts/gpu/parity_sweep.py > gpurun_out/sweep10.jsonl 2> gpurun_out/sweep10.err; echo "sweep rc=$?"
cut -c1-200 gpurun_out/sweep10.jsonl
