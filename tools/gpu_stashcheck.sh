timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_q.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest_q.log; tail -2 gpurun_out/pytest_q.log
for a in "alexnet bs t3" "m1 bs uniform" "vgg16 hybrid gaussian" "m1 bs t3"; do ITERS=30 python tools/stash_diag.py $a 2>&1 | grep -v "^  it" | grep -v "^l [0-9] \|^l1[0-1]" | tail -6; done
NOTEST=1 REPS=1 BENCH_ARGS="--workload alexnet --policy bs --dist t3" bash tools/gpu_ab.sh default
NOTEST=1 REPS=1 BENCH_ARGS="--workload m1 --policy bs --dist uniform" bash tools/gpu_ab.sh default
NOTEST=1 REPS=1 BENCH_ARGS="--workload m1 --policy bs --dist t3" bash tools/gpu_ab.sh default
NOTEST=1 REPS=2 bash tools/gpu_ab.sh default
