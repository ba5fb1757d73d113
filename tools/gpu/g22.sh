D=gpurun_out/g22
mkdir -p $D
for rep in 1 2 3; do for t in "32,16,0,8,6" "32,16,0,8,3" "32,16,4,8,6" "32,16,4,8,3"; do for wl in vgg16 m1; do
  RGC_TUNE=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$t $wl', round(d['value'],4), round(d['roofline']['achieved']), {k:round(v,4) for k,v in d['phase_ms'].items() if k in ('count_search','compact')})" >> $D/ab.txt 2>&1
done; done; done
sort $D/ab.txt
