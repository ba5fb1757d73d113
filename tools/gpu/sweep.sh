# measurement sweep over BASELINE.json's configs at N = $NG GPUs:
# one bench line per (workload, policy, dist); output $D/*.json
NG=${NG:-1}
D=gpurun_out/sweep_${NG}${TAG:-}
mkdir -p $D
port=29600
run() {  # name args...
  name=$1; shift
  port=$((port+1))
  if [ "$NG" = 1 ]; then
    timeout 400 python bench.py --no-cpu-baseline --no-e2e ${EXTRA:-} "$@" > $D/$name.json 2> $D/$name.err
  else
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $port bench.py --gpus $NG --no-cpu-baseline --no-e2e ${EXTRA:-} "$@" > $D/$name.json 2> $D/$name.err
  fi
  python -c "import json; d=json.load(open('$D/$name.json')); print('$name', round(d['value'],4), 'compress GB/s', round(d['compress_GBps_per_gpu']), 'K1 frac', round(d['roofline']['frac'],3), 'ag GB/s', d['allgather']['GBps_per_rank'], {k:round(v,4) for k,v in d['phase_ms'].items()})" || tail -3 $D/$name.err
}
run c1 --workload c1 --policy trimmed
run c1_bs --workload c1 --policy bs
run resnet50 --workload resnet50
run vgg16 --workload vgg16
run vgg16_bs --workload vgg16 --policy bs
run vgg16_trimmed --workload vgg16 --policy trimmed
run alexnet_bs_t3 --workload alexnet --policy bs --dist t3
run lstm_ptb --workload lstm_ptb
run lstm_wiki2 --workload lstm_wiki2
if [ "$NG" = 1 ]; then
run m1_trimmed --workload m1 --policy trimmed
run m1_bs --workload m1 --policy bs
run m1_bs_t3 --workload m1 --policy bs --dist t3
run m1_bs_uniform --workload m1 --policy bs --dist uniform
fi
