D=gpurun_out/g12
mkdir -p $D
CMD="python tools/decbench.py"
TAB=1 PS=4 timeout 300 $CMD > $D/plain.txt 2>&1 && TAB=1 PS=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_scatter" -s 6 -c 3 -o $D/dec -f $CMD > $D/ncu.log 2>&1; echo "ncu_rc=$?" >> $D/ncu.log
tail -3 $D/ncu.log
