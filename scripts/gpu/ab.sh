# A/B of raster variants at a config (stage times); usage: CFG=c4 bash scripts/gpu/ab.sh v1 v2 ...
mkdir -p gpurun_out
CFG=${CFG:-c4}
for v in "$@"; do
  if [ "$v" = cur ]; then d=.; else d=_ab/$v; fi
  extra=""; grep -q no-secondary $d/bench.py && extra="--no-secondary"
  (cd $d && timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $extra > $GRAFT_REPO_ROOT/gpurun_out/ab_$v.json 2> $GRAFT_REPO_ROOT/gpurun_out/ab_$v.err)
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value'],2), {k:v for k,v in d['extra']['stage_ms'].items() if v>0.01})" || tail -n 3 gpurun_out/ab_$v.err
done
