mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "asq" -x -p no:cacheprovider > gpurun_out/asq_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/asq_pytest.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e --asq > gpurun_out/bv_asq.json 2>gpurun_out/bv_asq.err
CMD="python bench.py --steps 5 --warmup 12 --no-cpu-baseline --no-e2e --asq"
timeout 300 $CMD > gpurun_out/it_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/asq_launches.csv $CMD > /dev/null 2>&1
tail -3 gpurun_out/asq_pytest.log
python -c "import json; d=json.load(open('gpurun_out/bv_asq.json')); print(d['value'], d['phase_ms'], d['message_bytes_per_rank'])"
python tools/launch_stats.py gpurun_out/asq_launches.csv
