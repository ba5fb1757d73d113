# parity (fast subset) of the default build, then bench + K2/K3 launch times per variant
# usage: bash tools/gpu_var.sh default w16 ...   (variant libs from tools/mkvar.sh)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
for v in "$@"; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-phase-events > gpurun_out/bv_$v.json 2>gpurun_out/bv_$v.err
  CMD="python bench.py --steps 5 --warmup 12 --no-cpu-baseline --no-e2e"
  timeout 300 $CMD > gpurun_out/pl_$v.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_count|k3_compact|k1_acc|k6_dec" --csv --log-file gpurun_out/l_$v.csv $CMD > /dev/null 2>&1
done
echo done
