# fill forked after K2 together with 512-thread K45 CTAs that fit beside a fill CTA
D=gpurun_out/g25
mkdir -p $D
for rep in 1 2; do for v in "default 1" "default 2" "k45_512 1" "k45_512 2" "k45_512b 2"; do set -- $v; for wl in vgg16 resnet50 m1; do
  if [ "$1" = default ]; then export RGC_LIB_PATH=; else export RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_$1.so; fi
  RGC_FILL_AT=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload $wl > $D/ab.json 2>$D/ab.err
  python -c "import json; d=json.load(open('$D/ab.json')); print('$1 at$2 $wl', round(d['value'],4))" >> $D/ab.txt 2>&1
done; done; done
export RGC_LIB_PATH=
RGC_LIB_PATH=$PWD/paper_1808_04357_b200/librgc_k45_512.so RGC_FILL_AT=2 timeout 300 python tools/timeline.py --workload vgg16 > $D/tl.json 2>&1
sort $D/ab.txt; python -c "import json; d=json.load(open('$D/tl.json')); print(d['step_us_median']); [print(k, round(v['start_us'],1), round(v['end_us'],1)) for k,v in d['timeline'].items()]"
