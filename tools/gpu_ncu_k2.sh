mkdir -p gpurun_out
./tools/readbw > gpurun_out/readbw.log 2>&1
export RGC_LIB_PATH=${K2LIB:-}
CMD="python bench.py --steps 3 --warmup 12 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/nk_plain.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k2_count" --launch-skip 20 -c 1 -o gpurun_out/k2_full -f $CMD > gpurun_out/nk_ncu.log 2>&1
echo done
