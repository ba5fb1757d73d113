# one development iteration on the GPU box: parity suite (fast subset), bench lines,
# and the per-kernel launch list of a short bench run (ncu only after a clean run)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bv_default.json 2>gpurun_out/bv_default.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-phase-events > gpurun_out/bv_noev.json 2>gpurun_out/bv_noev.err
CMD="python bench.py --steps 5 --warmup 12 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/it_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_launches.csv $CMD > /dev/null 2>&1
echo done
