# multi-GPU check on $NG GPUs: the NCCL/P2P/PULL parity worker + status scenarios, and the bench line
NG=${NG:-2}
D=gpurun_out/${TAG:-mgpu}
mkdir -p $D
nvidia-smi topo -m > $D/topo.txt 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider -rA > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $NG ${BENCH_ARGS:-} > $D/bench_n$NG.json 2> $D/bench_n$NG.err; echo "bench_rc=$?" >> $D/bench_n$NG.err
tail -5 $D/pytest.log; head -c 400 $D/bench_n$NG.json
