# final-build sanity on one GPU: smoke, the whole -m gpu suite, the default bench line
D=gpurun_out/final_sanity
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; echo "smoke_rc=$?" >> $D/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; echo "bench_rc=$?" >> $D/bench.err
tail -n 2 $D/smoke.log; tail -n 2 $D/pytest.log; head -c 300 $D/bench.json
if [ -n "$SWEEP" ]; then NG=1 TAG=_final2 bash tools/gpu/sweep.sh > $D/sweep.txt 2>&1; cut -c1-120 $D/sweep.txt; fi
if [ -n "$TL" ]; then for wl in vgg16 m1 resnet50 c1; do timeout 300 python tools/timeline.py --workload $wl > $D/timeline_$wl.json 2>&1; done; fi
