# multi-GPU: NCCL/P2P parity tests + bench lines at N = $NG for each sync mode (gpurun --gpus $NG)
mkdir -p gpurun_out
NG=${NG:-2}
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider > gpurun_out/mgpu_pytest_$NG.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/mgpu_pytest_$NG.log
port=29541
for m in ${MODES:-fixed p2p}; do
  port=$((port+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $port bench.py --gpus $NG --sync-mode $m --no-e2e > gpurun_out/mbench_${m}_$NG.json 2> gpurun_out/mbench_${m}_$NG.err
  echo "rc=$?" >> gpurun_out/mbench_${m}_$NG.err
done
echo done
