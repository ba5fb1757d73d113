"""Decompression of p simulated ranks' VGG16 messages on one GPU (development tool):
times the full rank-ordered K6 path and the prefill path (fill + scatter).  TAB=1: the
messages carry their producer range tables (k_tab) and the decompression reads them
(RGC_ASSUME_TAB), as between multi-rank contexts; otherwise k6_prep derives the ranges."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1808_04357_b200 import rgc as R

specs, sizes, _ = bench.layer_specs("vgg16", "hybrid", "--asq" in sys.argv)
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(5)
P = [int(x) for x in os.environ.get("PS", "1,2,4,8").split(",")]
TAB = os.environ.get("TAB") == "1"
one = R.RGC(specs, nranks=max(P) if TAB and max(P) > 1 else 1, device=0)
V = [torch.zeros(n, device=dev) for n in sizes]
U = [torch.zeros(n, device=dev) for n in sizes]
blocks = []
for i in range(max(P) + 6):
    one.compress([torch.randn(n, device=dev, generator=gen) * 0.01 for n in sizes], V, U)
    if i >= 6:
        blocks.append(one.msg.clone())
one.close()
out = [torch.empty(n, device=dev) for n in sizes]
for p in P:
    if TAB:
        os.environ["RGC_ASSUME_TAB"] = "1"
    eng = R.RGC(specs, nranks=p, device=0)
    os.environ.pop("RGC_ASSUME_TAB", None)
    eng.gathered.copy_(torch.cat(blocks[:p]) if p > 1 else blocks[0])
    for mode in ("full", "prefill"):
        def f():
            if mode == "prefill":
                eng.prefill_outputs(out)
            eng.decompress(out)
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        ts = []
        for _ in range(15):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); f(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        extra = ""
        if os.environ.get("RGC_TIMELINE") == "1":   # the scatter kernel alone (first start .. last exit)
            sc = []
            for _ in range(5):
                f(); torch.cuda.synchronize()
                tl = R.rgc_debug_timeline(eng.ctx)
                if "scatter" in tl:
                    sc.append(tl["scatter"][1] - tl["scatter"][0])
            if sc:
                extra = f"  scatter {statistics.median(sc):.1f} us"
        print(f"p={p} tab={int(TAB)} {mode}: {statistics.median(ts)*1e3:.1f} us{extra}", flush=True)
    eng.close()
