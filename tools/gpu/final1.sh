# final 1-GPU campaign: smoke, the -m gpu suite (default and checked builds), bench line +
# reference arm, sweep, ncu launch list + full captures (each after a clean run of the same command)
D=gpurun_out/final1
mkdir -p $D
nproc > $D/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $D/host.txt; nvidia-smi -q | grep -E "Product Name|Driver Version" >> $D/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $D/smoke.log 2>&1; echo "smoke_rc=$?" >> $D/smoke.log
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/pytest.log 2>&1; echo "pytest_rc=$?" >> $D/pytest.log
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_checked.so timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > $D/pytest_checked.log 2>&1; echo "pytest_rc=$?" >> $D/pytest_checked.log
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; echo "bench_rc=$?" >> $D/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 2 > $D/bench_reference.json 2> $D/bench_reference.err
NG=1 TAG=_final bash tools/gpu/sweep.sh > $D/sweep.txt 2>&1
for wl in vgg16 resnet50 m1 c1; do timeout 300 python tools/timeline.py --workload $wl > $D/timeline_$wl.json 2>&1; done
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > $D/plain.json 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $CMD > $D/ncu_list.log 2>&1; echo "ncu_list_rc=$?" >> $D/ncu_list.log
CMD2="python bench.py --steps 4 --warmup 10 --no-cpu-baseline --no-e2e"
timeout 300 $CMD2 > $D/plain2.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_acc|k2_stash|k3_compact|k45_cluster|k6_" -s 80 -c 9 -o $D/vgg16_full -f $CMD2 > $D/ncu_vgg16.log 2>&1; echo "ncu_rc=$?" >> $D/ncu_vgg16.log
CMD3="python bench.py --steps 4 --warmup 10 --no-cpu-baseline --no-e2e --workload m1 --policy bs"
timeout 300 $CMD3 > $D/plain3.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_acc|k2_stash|k3_compact|k6_" -s 60 -c 6 -o $D/m1_full -f $CMD3 > $D/ncu_m1.log 2>&1; echo "ncu_rc=$?" >> $D/ncu_m1.log
tail -n 1 $D/smoke.log; tail -n 2 $D/pytest.log; tail -n 2 $D/pytest_checked.log; head -c 400 $D/bench.json; echo; head -c 300 $D/bench_reference.json; echo; cat $D/sweep.txt | cut -c1-200; for f in ncu_list ncu_vgg16 ncu_m1; do tail -n 1 $D/$f.log; done
