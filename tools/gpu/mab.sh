# multi-GPU A/B: bench at N=$NG with env settings (e.g. RGC_NO_PAIRS=1) x sync modes
NG=${NG:-4}; port=29700
for rep in 1 2; do
for env in "X=0" "RGC_NO_PAIRS=1"; do
for m in ${MODES:-p2p pull}; do
  port=$((port+1))
  env $env timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $port bench.py --gpus $NG --no-cpu-baseline --no-e2e --sync-mode $m ${BENCH_ARGS:-} > gpurun_out/mab.json 2> gpurun_out/mab.err
  python -c "import json; d=json.load(open('gpurun_out/mab.json')); print('$env $m', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" || tail -3 gpurun_out/mab.err
done; done; done
