mkdir -p gpurun_out
timeout 1500 python scripts/parity_report.py c4 > gpurun_out/parity4.jsonl 2> gpurun_out/parity4.err; echo "parity rc=$?"
python - <<'P'
import json
for l in open('gpurun_out/parity4.jsonl'):
    d=json.loads(l)
    print(d['case'], d.get('error',''))
    if 'grads' in d:
        for k,v in d['grads'].items(): print('  ',k, round(v['max_ratio'],4), v['bad_rows'], v['worst_rows'], v['worst_vals'][0])
P
