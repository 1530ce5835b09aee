# frame base-offset sweep (BSR_CNT_SHIFT_KB, temporary A/B knob): stage times vs placement
CFG=${CFG:-c1}
for k in "$@"; do
  env BSR_CNT_SHIFT_KB=$k timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/sw.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sw.json')); s=d['extra']['stage_ms']; print('$CFG shift $k', round(d['value'],2), 'pre', s['preprocess'], 'scat', s['bin_scatter'], 'sort', s['tile_sort'], 'rfwd', s['raster_fwd'], 'rbwd', s['raster_bwd'], 'pbwd', s['preprocess_bwd'])"
done
