mkdir -p gpurun_out
for v in "default 1" "f32 1" "f32 2" "default 1" "f32 2"; do set -- $v
  if [ "$1" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$1.so; fi
  export RGC_FILL_AFTER=$2
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/b.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/b.json')); print('$1 after$2', round(d['value'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})"
done
