python scripts/gpu/exp_ulp.py
CFG=c4 bash scripts/gpu/ab.sh cur p4 p5 cur p4
CFG=c3 bash scripts/gpu/ab.sh cur p4
