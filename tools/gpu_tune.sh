# stash / bounded-histogram policy sweep (RGC_TUNE="F,min_margin,R,max_shift"): diag + bench per setting
mkdir -p gpurun_out
for t in ${TUNES:-6,2,3,10}; do
  RGC_TUNE=$t ITERS=60 python tools/stash_diag.py > gpurun_out/diag_$t.log 2>&1
  echo "TUNE $t" >> gpurun_out/tune.log
  tail -4 gpurun_out/diag_$t.log >> gpurun_out/tune.log
  RGC_TUNE=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/tb.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/tb.json')); print(round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> gpurun_out/tune.log
done
