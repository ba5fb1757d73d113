mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --maxfail=15 -p no:cacheprovider > gpurun_out/pytest1.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/pytest1.log
timeout 300 python tools/kbench.py --model vgg16 > gpurun_out/kb_vgg.log 2>&1
timeout 300 python tools/kbench.py --model m1 --policy trimmed > gpurun_out/kb_m1t.log 2>&1
timeout 300 python tools/kbench.py --model m1 --policy bs > gpurun_out/kb_m1b.log 2>&1
tail -5 gpurun_out/pytest1.log
