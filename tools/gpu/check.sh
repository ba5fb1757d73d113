# round-end style check on one GPU: smoke(), the whole -m gpu suite, the default bench line
D=gpurun_out/${TAG:-check}
mkdir -p $D
timeout 300 python __graft_entry__.py smoke > $D/smoke.log 2>&1; echo "smoke_rc=$?" >> $D/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider ${PYTEST_ARGS:-} > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
timeout 600 python bench.py > $D/bench.json 2> $D/bench.err; echo "bench_rc=$?" >> $D/bench.err
tail -5 $D/pytest.log; tail -2 $D/smoke.log; head -c 600 $D/bench.json
