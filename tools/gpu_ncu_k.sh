# full ncu capture of selected kernels (regex in $KRE) of a short bench run, after a clean run
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 12 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/nk_plain.log 2>&1 && timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"$KRE" --launch-skip ${SKIP:-30} -c ${CNT:-3} -o gpurun_out/${OUT:-kfull} -f $CMD > gpurun_out/nk_ncu.log 2>&1
echo done
