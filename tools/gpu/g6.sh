# A/B: where the decompression's zero fill is forked (RGC_FILL_AT=1 after K1, 2 after K2)
D=gpurun_out/g6
mkdir -p $D
RGC_FILL_AT=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_modes.py -q -m gpu -x -p no:cacheprovider -k "prefill or sync_mode or stash" > $D/pytest_at2.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_at2.log
for rep in 1 2 3; do for at in 1 2; do for wl in vgg16 resnet50 m1; do
  RGC_FILL_AT=$at timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('at$at $wl', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done; done
tail -2 $D/pytest_at2.log; cat $D/ab.txt
