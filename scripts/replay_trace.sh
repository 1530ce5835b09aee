# per-round clock64 trace of the fp64 forward replay (debug build of replay.cu only)
touch paper_2501_18630_b200/csrc/replay.cu
make -C paper_2501_18630_b200/csrc EXTRA=-DBSR_REPLAY_TRACE > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python bench.py --config c1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager 2>&1 | grep "^replay" | tail -80
