mkdir -p gpurun_out
for v in o3 o1; do
  if [ $v = o3 ]; then export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc.so; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_o1.so; fi
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_$v.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_$v.log
  timeout 300 python tools/kbench.py --model vgg16 > gpurun_out/kb_vgg_$v.log 2>&1
  timeout 300 python tools/kbench.py --model m1 --policy bs > gpurun_out/kb_m1b_$v.log 2>&1
done
