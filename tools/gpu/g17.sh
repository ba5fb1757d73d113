D=gpurun_out/g17
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2; do for v in coop nocoop; do for cfg in "vgg16 hybrid" "vgg16 trimmed" "m1 trimmed" "c1 trimmed" "resnet50 hybrid"; do set -- $cfg
  if [ "$v" = nocoop ]; then export RGC_NO_COOP_K4=1; else unset RGC_NO_COOP_K4; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $1 --policy $2 > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$v $1 $2', round(d['value'],4), d['gpu_launches'], {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done; done
unset RGC_NO_COOP_K4
tail -2 $D/pytest.log; cat $D/ab.txt
