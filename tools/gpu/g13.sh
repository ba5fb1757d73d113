# bucketed step (--buckets 2): A/B against the single context, K1 CTAs/SM of the big bucket
D=gpurun_out/g13
mkdir -p $D
for rep in 1 2; do
for cfg in "1 0" "2 3" "2 2" "2 1"; do set -- $cfg
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --buckets $1 --k1-occ-big $2 > $D/ab.json 2>$D/ab_$1_$2.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('buckets $1 occ $2', round(d['value'],4), round(d['roofline']['frac'],3), {k:round(v,4) for k,v in d['phase_ms'].items()})" >> $D/ab.txt 2>&1
done; done
tail -3 $D/ab_2_2.err; cat $D/ab.txt
