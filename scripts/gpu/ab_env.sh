# A/B of environment settings on the current tree: CFG=c4 bash scripts/gpu/ab_env.sh "BSR_RASTER_PX=1" "BSR_RASTER_PX=2"
mkdir -p gpurun_out
CFG=${CFG:-c4}
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/abe_$i.json 2> gpurun_out/abe_$i.err
  python -c "
import json,sys; d=json.load(open('gpurun_out/abe_$i.json')); print('$e', round(d['value'],2), {k:v for k,v in d['extra']['stage_ms'].items() if v>0.005})" || tail -n 3 gpurun_out/abe_$i.err
done
