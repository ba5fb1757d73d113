D=gpurun_out/g7
mkdir -p $D
for rep in 1 2; do
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k3a3.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "test_single_layer_sizes" > $D/k3a3_$rep.log 2>&1; echo "rc=$?" >> $D/k3a3_$rep.log
done
RGC_SYNC_EACH=1 RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k3a3.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider -k "test_single_layer_sizes" > $D/k3a3_sync.log 2>&1; echo "rc=$?" >> $D/k3a3_sync.log
for f in $D/k3a3_*.log; do echo "== $f"; grep -E "rgc error|passed|failed|rc=" $f | head -5; done
