python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/pytest_gpu13.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/pytest_gpu13.log
CFG=c4 bash scripts/gpu/ab.sh cur old cur old
CFG=c3 bash scripts/gpu/ab.sh cur old
CFG=c1 bash scripts/gpu/ab.sh cur old
python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -k "c1 or c4-0-True-0" > gpurun_out/pytest_gpu13b.log 2>&1; echo "fullsize rc=$?"; tail -2 gpurun_out/pytest_gpu13b.log
