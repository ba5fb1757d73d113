D=gpurun_out/g26
mkdir -p $D
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_sc4.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2 3; do for v in default sc4; do for wl in vgg16 resnet50 m1; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$v $wl', round(d['value'],4), round(d['phase_ms']['decompress'],4))" >> $D/ab.txt 2>&1
done; done; done
export RGC_LIB_PATH=
tail -2 $D/pytest.log; sort $D/ab.txt
