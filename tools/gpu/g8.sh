# 4 GPUs: multi-GPU worker (2 and 4 ranks), bench N=4 (push) with and without producer tables
D=gpurun_out/g8
mkdir -p $D
nvidia-smi topo -m > $D/topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -rA > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for rep in 1 2; do for v in tab notab; do
  if [ "$v" = notab ]; then export RGC_NO_TAB=1; else unset RGC_NO_TAB; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700+rep)) bench.py --gpus 4 --no-cpu-baseline --no-e2e > $D/ab_$v.json 2> $D/ab_$v.err
  python -c "import json; d=json.load(open('$D/ab_$v.json')); print('$v', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done
unset RGC_NO_TAB
tail -4 $D/pytest.log; cat $D/ab.txt
