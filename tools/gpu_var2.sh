mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1_parity or prefill_fill or mixed or asq_sizes" -p no:cacheprovider > gpurun_out/pv_$v.log 2>&1; echo "$v pytest_rc=$?"
  for r in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b_$v.json')); print('$v', round(d['value'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
  done
done
