# N-GPU: parity tests, bench lines (p2p plain / fixed / p2p asq), calibration
mkdir -p gpurun_out
NG=${NG:-4}
timeout 900 python -m pytest tests/test_multigpu.py -q -m gpu -p no:cacheprovider > gpurun_out/mgpu_pytest_$NG.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/mgpu_pytest_$NG.log
port=29641
for v in "p2p" "fixed" "p2p --asq"; do
  port=$((port+1)); tag=$(echo $v | tr -d ' -')
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $port bench.py --gpus $NG --sync-mode $v --no-e2e > gpurun_out/mb_${tag}_$NG.json 2> gpurun_out/mb_${tag}_$NG.err
done
port=$((port+1))
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port $port tools/calibrate.py --out gpurun_out/calib_$NG.json > gpurun_out/calib_$NG.log 2>&1
tail -n 3 gpurun_out/mgpu_pytest_$NG.log
for f in gpurun_out/mb_*_$NG.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['value'],4), {k: round(v,4) for k,v in d['phase_ms'].items()})" || tail -n 5 ${f%.json}.err; done
python -c "import json; d=json.load(open('gpurun_out/calib_$NG.json')); print(d['fit'], d['step'], d['dense_allreduce'])"
