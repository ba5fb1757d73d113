# prefill development iteration: new parity tests, quick parity suite, bench lines, launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "prefill" -x -p no:cacheprovider > gpurun_out/pf_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pf_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow and not prefill" --maxfail=5 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bv_default.json 2>gpurun_out/bv_default.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-phase-events > gpurun_out/bv_noev.json 2>gpurun_out/bv_noev.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e --graph --pool 4 > gpurun_out/bv_graph.json 2>gpurun_out/bv_graph.err
CMD="python bench.py --steps 5 --warmup 12 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/it_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/it_launches.csv $CMD > /dev/null 2>&1
tail -3 gpurun_out/pf_pytest.log; tail -3 gpurun_out/pytest_q.log; cat gpurun_out/smoke.log
for f in bv_default bv_noev bv_graph; do python -c "import json,sys; d=json.load(open('gpurun_out/$f.json')); print('$f', d['value'], d['phase_ms'])"; done
