# zero-fill width sweep (RGC_FILL_CTAS active issuing CTAs) on the default bench
for rep in 1 2; do for n in ${NS:-148 96 64 40}; do
  RGC_FILL_CTAS=$n timeout 300 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/fc.json 2>gpurun_out/fc.err
  python -c "import json; d=json.load(open('gpurun_out/fc.json')); print('ctas $n', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" || tail -3 gpurun_out/fc.err
done; done
