mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu3.log
timeout 1500 python scripts/parity_report.py needle c3 c3:17 c4 > gpurun_out/parity3.jsonl 2> gpurun_out/parity3.err; echo "parity rc=$?"
python - <<'P'
import json
for l in open('gpurun_out/parity3.jsonl'):
    d=json.loads(l)
    print(d['case'], d.get('error',''))
    if 'grads' in d:
        for k,v in d['grads'].items(): print('  ',k, round(v['max_ratio'],4), v['bad_rows'], v['worst_rows'])
    elif 'forward' not in d:
        print({k:v for k,v in d.items() if k!='case'})
P
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err; echo "bench rc=$?"
cut -c1-2500 gpurun_out/bench_c1.json
