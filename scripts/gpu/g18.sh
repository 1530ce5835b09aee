mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b18.json 2> gpurun_out/b18.err; echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/b18.json')); print(d['value'], d['e2e']['value'], d['extra']['e2e_graph']['value']); s=d['secondary']['c1']; print(s['value'], s['e2e']['value'], s['e2e_graph']['value'])"
tail -3 gpurun_out/b18.err
