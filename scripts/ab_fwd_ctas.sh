# A/B: raster_fwd register budget (BSR_FWD_CTAS resident CTAs per SM)
for V in 3 4; do
  touch paper_2501_18630_b200/csrc/raster_fwd.cu
  make -C paper_2501_18630_b200/csrc EXTRA="-DBSR_FWD_CTAS=$V" > /dev/null 2>&1 || { echo build failed; exit 1; }
  for C in c1 c3 c4; do
    S=50; [ $C = c3 ] && S=3; [ $C = c4 ] && S=10
    timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ctas=$V $C', round(d['value'],1), 'fwd', d['extra']['stage_ms']['raster_fwd'])"
  done
done
