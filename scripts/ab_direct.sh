# A/B: raster_bwd direct-atomics threshold (BSR_BWD_DIRECT_MAX)
for V in 1 2 3 5; do
  for C in c1 c3 c4; do
    S=50; [ $C = c3 ] && S=3; [ $C = c4 ] && S=10
    BSR_BWD_DIRECT=$V timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_x.json 2>/dev/null
    python3 -c "import json; d=json.loads(open('gpurun_out/ab_x.json').read().strip().splitlines()[-1]); s=d['extra']['stage_ms']; print('direct=$V $C', round(d['value'],1), s['raster_bwd'])"
  done
done
