for rep in 1 2; do for F in 6 4 3; do
 for wl in "--workload vgg16" "--workload alexnet --policy bs --dist t3"; do
  RGC_TUNE=32,16,0,8,$F timeout 300 python bench.py --no-cpu-baseline --no-e2e $wl > gpurun_out/f.json 2>gpurun_out/f.err
  python -c "import json; d=json.load(open('gpurun_out/f.json')); print('F $F', '$wl'[11:18], round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items() if k in ('count_search','compact')})"
 done; done; done
