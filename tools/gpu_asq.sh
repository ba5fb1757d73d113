# ASQ development iteration: ASQ + prefill parity, the quick parity suite, smoke, a bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "asq" -x -p no:cacheprovider > gpurun_out/asq_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/asq_pytest.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow and not asq" --maxfail=3 -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bv_default.json 2>gpurun_out/bv_default.err
tail -25 gpurun_out/asq_pytest.log; tail -3 gpurun_out/pytest_q.log; tail -2 gpurun_out/smoke.log
python -c "import json; d=json.load(open('gpurun_out/bv_default.json')); print(d['value'], d['phase_ms'])"
