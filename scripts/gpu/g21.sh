mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_suite.py -q -x > gpurun_out/pytest21.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest21.log
for c in c2 c1; do timeout 900 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b21_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b21_$c.json')); print('$c', d['value'], d['e2e']['value'], d['extra'].get('e2e_graph',{}).get('value'))"; done
