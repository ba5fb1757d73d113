mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 12 --no-cpu-baseline --no-e2e --asq"
timeout 300 $CMD > gpurun_out/nk_plain.log 2>&1 && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k5_asq|k2_stash|k3_compact" --launch-skip 36 -c 4 -o gpurun_out/asq_full -f $CMD > gpurun_out/nk_ncu.log 2>&1
echo rc=$?
