# ncu --set full (with source) of the warm VGG16 step's selection kernels and K1, plus the
# per-launch list; each ncu after the same command exited 0 without ncu
D=gpurun_out/${TAG:-prof}
mkdir -p $D
CMD="python bench.py --steps 4 --warmup 10 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-}"
timeout 300 $CMD > $D/plain.json 2> $D/plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k2_stash|k3_compact|k45_cluster|k1_acc}" -s ${SKIP:-55} -c ${COUNT:-6} -o $D/full -f $CMD > $D/ncu_full.log 2>&1; echo "ncu_full_rc=$?" >> $D/ncu_full.log
timeout 300 $CMD > $D/plain2.json 2> $D/plain2.err && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/launches.csv $CMD > $D/ncu_list.log 2>&1; echo "ncu_list_rc=$?" >> $D/ncu_list.log
tail -2 $D/ncu_full.log $D/ncu_list.log
