D=gpurun_out/g23
mkdir -p $D
for wl in "vgg16 hybrid" "resnet50 hybrid" "m1 bs" "c1 trimmed"; do set -- $wl
  timeout 300 python tools/timeline.py --workload $1 --policy $2 > $D/tl_$1_$2.json 2> $D/tl_$1_$2.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
tail -2 $D/pytest.log; cat $D/tl_vgg16_hybrid.json
