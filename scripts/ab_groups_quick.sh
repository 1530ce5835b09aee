for G in 4 2; do
  for C in c1 c3 c4; do
    S=50; [ $C = c3 ] && S=3; [ $C = c4 ] && S=10
    BSR_RASTER_G=$G timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_g.json 2>/dev/null
    python3 -c "import json; d=json.loads(open('gpurun_out/ab_g.json').read().strip().splitlines()[-1]); s=d['extra']['stage_ms']; print('G=$G $C', round(d['value'],1), s['raster_fwd'], s['raster_bwd'])"
  done
done
