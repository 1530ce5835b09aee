mkdir -p gpurun_out
for i in 1 2 3; do
for P in 0 1; do
  BSR_NO_PDL=$P timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/pdl_$P.json 2>/dev/null
  python3 -c "import json;d=json.loads(open('gpurun_out/pdl_$P.json').read().strip().splitlines()[-1]);print('NO_PDL=$P', round(d['value'],1), round(d['ms_per_step'],4))"
done
done
