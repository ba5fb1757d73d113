# RGC_SYNC_P2P push kernel width (CTAs per destination) at N=$NG
NG=${NG:-2}; port=29900
for rep in 1 2; do for nb in ${NBS:-32 64 128}; do
  port=$((port+1))
  RGC_P2P_NB=$nb timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $port bench.py --gpus $NG --no-cpu-baseline --no-e2e > gpurun_out/nb.json 2> gpurun_out/nb.err
  python -c "import json; d=json.load(open('gpurun_out/nb.json')); print('nb $nb', round(d['value'],4), {k:round(v,4) for k,v in d['phase_ms'].items()})" || tail -3 gpurun_out/nb.err
done; done
