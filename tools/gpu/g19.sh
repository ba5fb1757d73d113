D=gpurun_out/g19
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2; do for v in hint nocoop; do for cfg in "vgg16 hybrid" "vgg16 trimmed" "m1 trimmed" "c1 trimmed" "resnet50 hybrid"; do set -- $v $cfg
  if [ "$1" = nocoop ]; then export RGC_NO_COOP_K4=1; else unset RGC_NO_COOP_K4; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $2 --policy $3 > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$1 $2 $3', round(d['value'],4), d['gpu_launches'], {k:round(v,4) for k,v in d['phase_ms'].items() if k in ('select','emit')})" >> $D/ab.txt 2>&1
done; done; done
tail -2 $D/pytest.log; sort $D/ab.txt
