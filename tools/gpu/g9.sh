D=gpurun_out/g9
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "tables or prefill or multi_layer" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
PS=2,4,8 timeout 300 python tools/decbench.py > $D/dec_notab.txt 2>&1
TAB=1 PS=2,4,8 timeout 300 python tools/decbench.py > $D/dec_tab.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $D/bench.json 2> $D/bench.err
tail -2 $D/pytest.log; cat $D/dec_notab.txt $D/dec_tab.txt; python -c "import json; d=json.load(open('$D/bench.json')); print(d['value'], d['roofline']['frac'], d['phase_ms'])"
