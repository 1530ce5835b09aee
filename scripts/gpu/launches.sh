# ncu launch list (gpu__time_duration per kernel, cold cache, serialised) of a bench command
mkdir -p gpurun_out
CFG=${CFG:-c4}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary"
$CMD > gpurun_out/launch_plain_$CFG.log 2>&1 || { echo plain failed; tail gpurun_out/launch_plain_$CFG.log; exit 1; }
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/launch_ncu_$CFG.log 2>&1
echo "ncu rc=$?"; wc -l gpurun_out/launches_$CFG.csv
