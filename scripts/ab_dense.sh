# A/B: raster dense-mode threshold (BSR_DENSE_X10 = 10 x groups per entry)
for V in 35 40 50; do
  touch paper_2501_18630_b200/csrc/raster_fwd.cu paper_2501_18630_b200/csrc/raster_bwd.cu
  make -C paper_2501_18630_b200/csrc EXTRA="-DBSR_DENSE_X10=$V" > /dev/null 2>&1 || { echo build failed; exit 1; }
  for C in c1 c3 c4; do
    S=50; [ $C = c3 ] && S=3; [ $C = c4 ] && S=10
    timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_d.json 2>/dev/null
    python3 -c "import json; d=json.loads(open('gpurun_out/ab_d.json').read().strip().splitlines()[-1]); s=d['extra']['stage_ms']; print('x10=$V $C', round(d['value'],1), s['raster_fwd'], s['raster_bwd'])"
  done
done
