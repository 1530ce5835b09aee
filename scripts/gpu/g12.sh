CFG=c4 bash scripts/gpu/ab.sh cur s6 u8 s6u8 s8 cur s6 s8
