# every bench line of the round: default (c4 + nested c1, CPU baselines), c2, c3, reference arm
mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02_default.json 2> gpurun_out/r02_default.err; echo "default rc=$?"
timeout 900 python bench.py --config c2 --steps 100 --warmup 5 > gpurun_out/r02_c2.json 2> gpurun_out/r02_c2.err; echo "c2 rc=$?"
timeout 1500 python bench.py --config c3 --steps 5 --warmup 3 > gpurun_out/r02_c3.json 2> gpurun_out/r02_c3.err; echo "c3 rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
for f in default c2 c3 ref; do python -c "
import json; d=json.load(open('gpurun_out/r02_$f.json')); print('$f', d['config'], d['value'], d.get('e2e',{}) and d['e2e']['value'], d.get('roofline',{}) and d['roofline'].get('frac'), d.get('cpu_baseline') and d['cpu_baseline'].get('value'))"; done
