mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_c1.json 2> gpurun_out/e2e_c1.err
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/e2e_c2.json 2> gpurun_out/e2e_c2.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:raster_ -s 6 -c 2 -o gpurun_out/raster_c1 $CMD > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu.log
cut -c1-300 gpurun_out/e2e_c1.json gpurun_out/e2e_c2.json
