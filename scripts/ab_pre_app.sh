for v in 128 0 128 0; do
  BSR_PRE_APP_BULK=$v timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value'],1), d['extra']['stage_ms']['preprocess'])"
done
for v in 128 0; do
  BSR_PRE_APP_BULK=$v timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 $v', round(d['value'],1), d['extra']['stage_ms']['preprocess'])"
done
