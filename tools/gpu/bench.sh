# one GPU call: bench line (+ reference arm), launch list, ncu --set full of one warm step
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo "ncu1_rc=$?" >> gpurun_out/ncu1.log
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_|k2_|k3_|k4_|k45|k5_|k6_" -s 60 -c 12 -o gpurun_out/prof_full -f $CMD > gpurun_out/ncu2.log 2>&1; echo "ncu2_rc=$?" >> gpurun_out/ncu2.log
cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'])"
tail -n 2 gpurun_out/ncu1.log; tail -n 2 gpurun_out/ncu2.log
