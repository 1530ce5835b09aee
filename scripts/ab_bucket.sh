# A/B: per-tile sort big-bucket threshold (BSR_MAX_BUCKET)
for V in 8 16 32; do
  touch paper_2501_18630_b200/csrc/bin.cu
  make -C paper_2501_18630_b200/csrc EXTRA="-DBSR_MAX_BUCKET=$V" > /dev/null 2>&1 || { echo build failed; exit 1; }
  for C in c1 c2 c3 c4; do
    S=50; [ $C = c2 ] && S=100; [ $C = c3 ] && S=3; [ $C = c4 ] && S=10
    timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_b.json 2>/dev/null
    python3 -c "import json; d=json.loads(open('gpurun_out/ab_b.json').read().strip().splitlines()[-1]); s=d['extra']['stage_ms']; print('maxb=$V $C', round(d['value'],1), s['tile_sort'])"
  done
done
