# A/B: preprocess eager appearance copy size limit (BSR_EAGER_APP_MAX_N)
for V in 2097152 100000000; do
  touch paper_2501_18630_b200/csrc/preprocess.cu
  make -C paper_2501_18630_b200/csrc EXTRA="-DBSR_EAGER_APP_MAX_N=$V" > /dev/null 2>&1 || { echo build failed; exit 1; }
  for C in c3 c4; do
    S=3; [ $C = c4 ] && S=10
    timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_e.json 2>/dev/null
    python3 -c "import json; d=json.loads(open('gpurun_out/ab_e.json').read().strip().splitlines()[-1]); s=d['extra']['stage_ms']; print('eager<=$V $C', round(d['value'],1), s['preprocess'])"
  done
done
