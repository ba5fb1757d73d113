mkdir -p gpurun_out
for v in e f a; do
  export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "not slow" -p no:cacheprovider > gpurun_out/var_${v}_pytest.log 2>&1
  for m in "vgg16 hybrid" "m1 bs" "m1 trimmed"; do set -- $m
    timeout 300 python tools/kbench.py --model $1 --policy $2 > gpurun_out/var_${v}_$1_$2.log 2>&1
  done
done
