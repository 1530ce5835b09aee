mkdir -p gpurun_out
S=$(date +%s); timeout 1150 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - S ))s"; tail -5 gpurun_out/pytest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
