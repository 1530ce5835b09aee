mkdir -p gpurun_out
cd oracle/_ref/pkg && PYTHONPATH=$GRAFT_REPO_ROOT/oracle/_ref/pkg:$GRAFT_REPO_ROOT/tests:$GRAFT_REPO_ROOT timeout 600 python -m pytest tests/test_rasterizer.py -q -rA -p ref_core_plugin -p no:cacheprovider -o addopts= > $GRAFT_REPO_ROOT/gpurun_out/refsuite.log 2>&1; echo "rc=$?"
cd $GRAFT_REPO_ROOT; grep -E "PASSED|FAILED|passed|failed|Error" gpurun_out/refsuite.log | tail -45
