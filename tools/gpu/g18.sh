D=gpurun_out/g18
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2; do for v in "coop1 1" "coop2 2" "coop4 4" "nocoop 0"; do set -- $v; for cfg in "vgg16 hybrid" "vgg16 trimmed" "m1 trimmed" "c1 trimmed"; do set -- $1 $2 $cfg
  if [ "$1" = nocoop ]; then export RGC_NO_COOP_K4=1; else unset RGC_NO_COOP_K4; export RGC_K4_COOP_OCC=$2; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $3 --policy $4 > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$1 $3 $4', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items() if k in ('select','emit')})" >> $D/ab.txt 2>&1
done; done; done
tail -2 $D/pytest.log; sort $D/ab.txt
