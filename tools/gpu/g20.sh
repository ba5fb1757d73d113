D=gpurun_out/g20
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "tables or prefill or multi_layer" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2; do TAB=1 PS=2,4,8 timeout 300 python tools/decbench.py >> $D/dec.txt 2>&1; done
tail -2 $D/pytest.log; cat $D/dec.txt
