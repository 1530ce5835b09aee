# A/B of the raster sub-warp group count (BSR_RASTER_G): parity first, then stage times
mkdir -p gpurun_out
for G in 4 2 1; do
  BSR_RASTER_G=$G timeout 240 python -m pytest tests -m gpu -x -q > gpurun_out/ab_pytest_G$G.log 2>&1
  echo "G=$G pytest: $(tail -1 gpurun_out/ab_pytest_G$G.log)"
done
for C in c1 c3 c4; do
  for G in 4 2 1; do
    S=30; [ $C = c1 ] && S=100
    [ $C = c3 ] && S=5
    BSR_RASTER_G=$G timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${C}_G$G.json 2> gpurun_out/ab_${C}_G$G.err
    python - "$C" "$G" <<'PY'
import json, sys
c, g = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/ab_{c}_G{g}.json").read().strip().splitlines()[-1])
    st = d["extra"]["stage_ms"]
    print(f"{c} G={g} value={d['value']:.1f} {d['unit']} raster_fwd={st['raster_fwd']:.4f} raster_bwd={st['raster_bwd']:.4f} frac={d['roofline']['frac']}")
except Exception as e:
    print(c, g, "failed", e)
PY
  done
done
