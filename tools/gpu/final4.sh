# final 4-GPU campaign: NVLink peak, the multi-GPU worker, bench lines at N = 2 and 4, cost model
D=gpurun_out/final4
mkdir -p $D
nvidia-smi topo -m > $D/topo.txt 2>&1
timeout 600 python tools/nvlink_bw.py --out $D/nvlink_peak.json > $D/nvlink.log 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -rA > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29800+n)) bench.py --gpus $n > $D/bench_n$n.json 2> $D/bench_n$n.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29810+n)) tools/calibrate.py --out $D/calibrate_n$n.json > $D/calibrate_n$n.log 2>&1
done
NG=4 TAG=_final4 bash tools/gpu/sweep.sh > $D/sweep4.txt 2>&1
tail -n 3 $D/pytest.log; grep peak $D/nvlink_peak.json; for n in 2 4; do head -c 250 $D/bench_n$n.json; echo; done; cat $D/sweep4.txt | cut -c1-160
