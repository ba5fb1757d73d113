D=gpurun_out/g1
mkdir -p $D
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/stream_bench tools/stream_bench.cu && timeout 300 tools/stream_bench > $D/stream_bench.json 2> $D/stream_bench.err
timeout 900 python tools/e2_sweep.py --sizes 16777216,100000000 --variants threshold_bs,sampled_bs --warm 3000 --out $D/e2_stationary.json > /dev/null 2> $D/e2_stationary.err
timeout 600 python tools/e2_sweep.py --sizes 16777216,100000000 --variants threshold_bs,sampled_bs --warm 10 --out $D/e2_drift.json > /dev/null 2> $D/e2_drift.err
TAG=g1/prof bash tools/gpu/prof.sh
cat $D/stream_bench.json; tail -3 $D/e2_stationary.err
