CFG=c4 bash scripts/gpu/ab.sh cur atom cur atom
