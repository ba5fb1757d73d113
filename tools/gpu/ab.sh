# A/B of library variants (tools/mkvar.sh): quick parity of the default build, then
# alternating bench runs per variant (value + phases)
# usage: bash tools/gpu_ab.sh default nohint ...   (REPS=2)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
tail -2 gpurun_out/pytest_q.log
fi
for rep in $(seq ${REPS:-2}); do
for v in "$@"; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$v', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})"
done
done
