# round-end style check: smoke, the whole -m gpu suite, the default bench line
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_all.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
tail -3 gpurun_out/pytest_all.log; cat gpurun_out/bench.json
