D=gpurun_out/g16
mkdir -p $D
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k3a3o1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider > $D/pytest_k3a3o1.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_k3a3o1.log
for rep in 1 2 3; do for v in default k3a3o1; do for wl in vgg16 resnet50; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$v $wl', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done; done
export RGC_LIB_PATH=
tail -2 $D/pytest_k3a3o1.log; cat $D/ab.txt
