D=gpurun_out/g2
mkdir -p $D
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu && timeout 400 tools/stream_bench 138342400 3 > $D/stream_bench.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider -k "sampled or nonfinite or degenerate or asq or stash" > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
timeout 900 python tools/e2_sweep.py --sizes 16777216,100000000 --variants threshold_bs,sampled_bs --warm 3000 --out $D/e2_stationary.json > /dev/null 2> $D/e2_stationary.err
timeout 300 python bench.py --no-cpu-baseline --no-e2e > $D/bench.json 2> $D/bench.err
tail -3 $D/pytest.log; cat $D/stream_bench.json; cat $D/e2_stationary.err | cut -c1-300; head -c 300 $D/bench.json
