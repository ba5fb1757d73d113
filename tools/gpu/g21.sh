D=gpurun_out/g21
mkdir -p $D
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2 3; do for v in default twobar; do for wl in vgg16 m1 resnet50; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$v $wl', round(d['value'],4), round(d['roofline']['achieved']), round(d['roofline']['frac'],4))" >> $D/ab.txt 2>&1
done; done; done
export RGC_LIB_PATH=
tail -2 $D/pytest.log; sort $D/ab.txt
