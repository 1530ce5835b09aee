# Full bench lines (all configs) + ncu launch list of the default command + ncu --set full of
# the top kernel; outputs under gpurun_out/
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/fb_c1.json 2> gpurun_out/fb_c1.err
for C in c2 c3 c4; do
  S=20; [ $C = c2 ] && S=100; [ $C = c3 ] && S=10
  timeout 600 python bench.py --config $C --steps $S --warmup 5 --no-cpu-baseline > gpurun_out/fb_$C.json 2> gpurun_out/fb_$C.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fb_ref.json 2> gpurun_out/fb_ref.err
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/fb_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fb_launches.csv $CMD > gpurun_out/fb_ncu1.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD2 > gpurun_out/fb_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:raster_(fwd|bwd)_kernel<0' -s 4 -c 2 -o gpurun_out/fb_raster_c1 $CMD2 > gpurun_out/fb_ncu2.log 2>&1
echo done
for f in gpurun_out/fb_c*.json gpurun_out/fb_ref.json; do cut -c1-200 $f; done
