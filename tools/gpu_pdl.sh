mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "not slow" -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
tail -2 gpurun_out/pytest_q.log
for v in pdl nopdl; do
  if [ $v = nopdl ]; then export RGC_NO_PDL=1; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b_$v.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --graph --pool 4 > gpurun_out/bg_$v.json 2>/dev/null
  for f in b_$v bg_$v; do python -c "import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"; done
done
