# A/B: forward replay CTA width (BSR_REPLAY_NT)
for C in c1 c3 c4; do
  for NT in 1024 256 128 64; do
    S=50; [ $C = c3 ] && S=3; [ $C = c4 ] && S=10
    BSR_REPLAY_NT=$NT timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_r.json 2>/dev/null
    python3 -c "import json; d=json.loads(open('gpurun_out/ab_r.json').read().strip().splitlines()[-1]); print('$C NT=$NT', round(d['value'],1), d['extra']['stage_ms']['replay_fwd'], d['extra']['flagged_pixels'])"
  done
done
