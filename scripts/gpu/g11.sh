mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --no-secondary --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['value'], d['roofline']['frac'], d['extra']['stage_ms'])"
tail -3 gpurun_out/bench_c4.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k needle > gpurun_out/needle.log 2>&1; tail -2 gpurun_out/needle.log
timeout 1500 python scripts/parity_report.py c4 > gpurun_out/parity11.jsonl 2> gpurun_out/parity11.err; echo "parity rc=$?"
python - <<'P'
import json
for l in open('gpurun_out/parity11.jsonl'):
    d=json.loads(l)
    print(d['case'], d.get('error',''), d.get('forward_ok'), d.get('grads_ok'))
    if 'grads' in d:
        for k,v in d['grads'].items(): print('  ',k, round(v['max_ratio'],4), v['bad_rows'], v.get('ill_posed_rows'), v['worst_rows'])
P
