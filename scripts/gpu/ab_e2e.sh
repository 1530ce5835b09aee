# A/B of the public-API (e2e) step: CFG=c4 bash scripts/gpu/ab_e2e.sh prev cur
mkdir -p gpurun_out
CFG=${CFG:-c4}
for v in "$@"; do
  if [ "$v" = cur ]; then d=.; else d=_ab/$v; fi
  (cd $d && timeout 600 python bench.py --config $CFG --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > $GRAFT_REPO_ROOT/gpurun_out/abe2e_$v.json 2>/dev/null)
  python -c "
import json; d=json.load(open('gpurun_out/abe2e_$v.json')); print('$CFG', '$v', round(d['value'],2), 'e2e', round(d['e2e']['value'],2))"
done
