# timing probe: how much of config 4's raster time the fp64 (unsafe) path costs
# (a build that classifies every primitive as fp32-safe; timing only, not exact)
touch paper_2501_18630_b200/csrc/preprocess.cu
make -C paper_2501_18630_b200/csrc EXTRA='-DBSR_UNSAFE_R2_ERR=1e30f' > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --config c4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('all-fp32', round(d['value'],1), d['extra']['stage_ms'], d['extra']['flagged_pixels'])"
