D=gpurun_out/g15
mkdir -p $D
timeout 300 python __graft_entry__.py smoke > $D/smoke.log 2>&1; echo "smoke_rc=$?" >> $D/smoke.log
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k3a3o1.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "test_single_layer_sizes or test_distributions" > $D/k3a3o1.log 2>&1; echo "rc=$?" >> $D/k3a3o1.log
tail -25 $D/pytest.log; tail -2 $D/smoke.log; tail -3 $D/k3a3o1.log
