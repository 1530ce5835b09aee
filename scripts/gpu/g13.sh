mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest13.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest13.log
CFG=c4 bash scripts/gpu/ab.sh cur
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c4 or c2" > gpurun_out/pytest13b.log 2>&1; echo "fullsize rc=$?"; tail -3 gpurun_out/pytest13b.log
