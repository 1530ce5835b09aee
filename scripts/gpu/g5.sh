mkdir -p gpurun_out
timeout 1500 python scripts/sensitivity.py c4 4892568 4863872 4843060 > gpurun_out/sens_c4.jsonl 2> gpurun_out/sens_c4.err; echo "rc=$?"
cat gpurun_out/sens_c4.jsonl; tail -3 gpurun_out/sens_c4.err
