mkdir -p gpurun_out/g0
nproc > gpurun_out/g0/host.txt; lscpu | head -20 >> gpurun_out/g0/host.txt
timeout 600 python bench.py > gpurun_out/g0/bench.json 2> gpurun_out/g0/bench.err; echo "bench_rc=$?" >> gpurun_out/g0/bench.err
CMD="python bench.py --workload m1 --policy bs --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/g0/m1.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_|k2_|k3_|k45|k6_" -s 30 -c 8 -o gpurun_out/g0/m1_full -f $CMD > gpurun_out/g0/ncu_m1.log 2>&1; echo "ncu_rc=$?" >> gpurun_out/g0/ncu_m1.log
tail -2 gpurun_out/g0/ncu_m1.log
