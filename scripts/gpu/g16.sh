mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest16.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest16.log
CFG=c4 bash scripts/gpu/ab_env.sh "BSR_RASTER_PX=1" "BSR_RASTER_PX=2"
CFG=c1 bash scripts/gpu/ab_env.sh "BSR_RASTER_PX=1" "BSR_RASTER_PX=2"
CFG=c3 bash scripts/gpu/ab_env.sh "BSR_RASTER_PX=1" "BSR_RASTER_PX=2"
