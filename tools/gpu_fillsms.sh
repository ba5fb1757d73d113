mkdir -p gpurun_out
for sms in 0 112 80 56 40; do
  export RGC_FILL_SMS=$sms
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --graph --pool 4 > gpurun_out/fs_g_$sms.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-phase-events > gpurun_out/fs_d_$sms.json 2>/dev/null
  for f in fs_g_$sms fs_d_$sms; do python -c "import json,sys; d=json.load(open(\"gpurun_out/$f.json\")); print(\"$f\", round(d[\"value\"],4), {k: round(v,4) for k,v in d[\"phase_ms\"].items()})"; done
done
