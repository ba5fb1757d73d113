D=gpurun_out/g24
mkdir -p $D
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2 3; do for v in coop nocoop; do for cfg in "vgg16 hybrid" "resnet50 hybrid" "m1 bs" "c1 trimmed" "alexnet bs"; do set -- $v $cfg
  if [ "$1" = nocoop ]; then export RGC_NO_COOP_K2=1; else unset RGC_NO_COOP_K2; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $2 --policy $3 > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$1 $2 $3', round(d['value'],4), d['gpu_launches'])" >> $D/ab.txt 2>&1
done; done; done
unset RGC_NO_COOP_K2
timeout 300 python tools/timeline.py --workload vgg16 > $D/tl_vgg16.json 2>&1
tail -2 $D/pytest.log; sort $D/ab.txt; head -50 $D/tl_vgg16.json
