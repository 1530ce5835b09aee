mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 profiles/micro/peaks.cu -o profiles/micro/peaks && python profiles/micro/run_peaks.py > gpurun_out/peaks.json 2>&1; cat gpurun_out/peaks.json
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
cut -c1-6000 gpurun_out/bench_default.json; tail -5 gpurun_out/bench_default.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
