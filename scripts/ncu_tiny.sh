# per-kernel durations of one graph-replayed training step at a tiny size (launch floor)
mkdir -p gpurun_out
python scripts/overhead_probe.py tiny > gpurun_out/tiny_plain.log 2>&1 || { echo plain failed; cat gpurun_out/tiny_plain.log; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tiny.csv \
    python scripts/overhead_probe.py tiny > gpurun_out/ncu_tiny.log 2>&1
echo "rc=$?"
