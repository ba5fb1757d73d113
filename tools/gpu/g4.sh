D=gpurun_out/g4
mkdir -p $D
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k3a3dbg.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "test_single_layer_sizes" -s > $D/k3dbg.log 2>&1; echo "rc=$?" >> $D/k3dbg.log
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k1s1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest_k1s1.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_k1s1.log
for rep in 1 2 3; do for v in default k1s1; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > $D/ab_$v.json 2>$D/ab_$v.err
  python -c "import json; d=json.load(open('$D/ab_$v.json')); print('$v', round(d['value'],4), round(d['roofline']['frac'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done
export RGC_LIB_PATH=
grep -E "K3 check|rc=|passed|failed" $D/k3dbg.log | head; tail -2 $D/pytest_k1s1.log; cat $D/ab.txt
