# parity (all gpu tests) + c1/c3/c4 stage times at the default raster config
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest: $(tail -1 gpurun_out/q_pytest.log)"
for C in c1 c3 c4; do
  S=30; [ $C = c1 ] && S=100; [ $C = c3 ] && S=5
  timeout 300 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q_$C.json 2> gpurun_out/q_$C.err
  python - "$C" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/q_{c}.json").read().strip().splitlines()[-1])
    st = d["extra"]["stage_ms"]
    print(c, f"value={d['value']:.1f} {d['unit']}", " ".join(f"{k}={v:.4f}" for k, v in st.items()), "flagged", d["extra"]["flagged_pixels"])
except Exception as e:
    print(c, "failed", e, open(f"gpurun_out/q_{c}.err").read()[-2000:])
PY
done
