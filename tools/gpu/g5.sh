# 2 GPUs: the whole GPU suite (1-GPU tests on device 0 + the 2-GPU worker), then A/B of the
# producer range tables (default) against receiver-side k6_prep (RGC_NO_TAB=1) at N = 2
D=gpurun_out/g5
mkdir -p $D
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2 3; do for v in tab notab; do
  if [ "$v" = notab ]; then export RGC_NO_TAB=1; else unset RGC_NO_TAB; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+rep)) bench.py --gpus 2 --no-cpu-baseline --no-e2e > $D/ab_$v.json 2> $D/ab_$v.err
  python -c "import json; d=json.load(open('$D/ab_$v.json')); print('$v', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done
unset RGC_NO_TAB
tail -3 $D/pytest.log; cat $D/ab.txt
