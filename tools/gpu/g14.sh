D=gpurun_out/g14
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2; do for v in default nosec; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  echo "== $v" >> $D/dec.txt
  TAB=1 PS=2,4,8 timeout 300 python tools/decbench.py >> $D/dec.txt 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$v', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done
export RGC_LIB_PATH=
tail -2 $D/pytest.log; cat $D/dec.txt $D/ab.txt
