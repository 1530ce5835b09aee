mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize.py > gpurun_out/pytest12.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest12.log
CFG=c4 bash scripts/gpu/ab.sh old cur
timeout 1500 python scripts/parity_report.py needle c3 c4 > gpurun_out/parity12.jsonl 2> gpurun_out/parity12.err; echo "parity rc=$?"
python - <<'P'
import json
for l in open('gpurun_out/parity12.jsonl'):
    d=json.loads(l)
    print(d['case'], d.get('error',''), d.get('forward_ok'), d.get('grads_ok'))
    if 'grads' in d:
        for k,v in d['grads'].items(): print('  ',k, round(v['max_ratio'],4), v['bad_rows'], v.get('ill_posed_rows'), v['worst_rows'])
    elif 'forward' not in d: print(d)
P
