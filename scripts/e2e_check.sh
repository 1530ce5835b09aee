mkdir -p gpurun_out
for C in c1 c2; do timeout 300 python bench.py --config $C --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_$C.json 2>/dev/null; python3 -c "import json;d=json.loads(open('gpurun_out/e2e_$C.json').read().strip().splitlines()[-1]);print('$C', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"; done
