# the round's profile set: new loss test, c4 launch list, ncu --set full of the raster and the other kernels
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "loss_both_tilings" > gpurun_out/pt_loss.log 2>&1; tail -1 gpurun_out/pt_loss.log
CFG=c4 bash scripts/gpu/launches.sh
bash scripts/gpu/ncu_c4.sh
bash scripts/gpu/ncu_c4_aux.sh
