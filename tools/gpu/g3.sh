D=gpurun_out/g3
mkdir -p $D
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu && timeout 400 tools/stream_bench 138342400 3 > $D/stream_bench.json 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest_default.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_default.log
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k3a3.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "not slow" > $D/pytest_k3a3.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_k3a3.log
for rep in 1 2 3; do for v in default k3a3; do
  if [ "$v" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > $D/ab_$v.json 2>$D/ab_$v.err
  python -c "import json; d=json.load(open('$D/ab_$v.json')); print('$v', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload resnet50 > $D/abr_$v.json 2>$D/abr_$v.err
  python -c "import json; d=json.load(open('$D/abr_$v.json')); print('r50 $v', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt
done; done
export RGC_LIB_PATH=
tail -2 $D/pytest_default.log $D/pytest_k3a3.log; cat $D/ab.txt; grep -E "u1|gs1_occ3|blk_occ3" $D/stream_bench.json
