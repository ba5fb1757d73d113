# A/B of K45 geometries: default (1024 threads, 176 KB keys, 1 CTA/SM) vs 256 / 512 threads
D=gpurun_out/g11
mkdir -p $D
for v in k45_256 k45_512; do
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest_$v.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_$v.log
done
for rep in 1 2; do for v in default k45_256 k45_512; do for wl in vgg16 resnet50; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$v $wl', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done; done
export RGC_LIB_PATH=
tail -1 $D/pytest_*.log; cat $D/ab.txt
