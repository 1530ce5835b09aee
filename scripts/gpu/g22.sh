mkdir -p gpurun_out
S=$(date +%s); timeout 1150 python -m pytest tests -m gpu -q -x > gpurun_out/pytest22.log 2>&1; echo "pytest rc=$? wall=$(( $(date +%s) - S ))s"; tail -3 gpurun_out/pytest22.log
CFG=c4 bash scripts/gpu/ab.sh prev cur; CFG=c1 bash scripts/gpu/ab.sh prev cur
