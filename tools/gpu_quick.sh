# parity suite + phase timing of the default build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
for m in "vgg16 hybrid" "m1 bs" "m1 trimmed"; do set -- $m
  timeout 300 python tools/kbench.py --model $1 --policy $2 > gpurun_out/q_$1_$2.log 2>&1
done
