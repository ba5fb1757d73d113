"""Per-step diagnostics of the BS layers of VGG16 (optionally ASQ): Alg.3 path, bounds, stash."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1808_04357_b200 import rgc as R

asq = "--asq" in sys.argv
specs, sizes, kinds = bench.layer_specs("vgg16", "hybrid", asq)
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(1)
G = [[torch.randn(n, device=dev, generator=gen) * 0.01 for n in sizes] for _ in range(6)]
V = [torch.zeros(n, device=dev) for n in sizes]
U = [torch.zeros(n, device=dev) for n in sizes]
O = [torch.empty(n, device=dev) for n in sizes]
eng = R.RGC(specs, device=0)
for it in range(16):
    eng.step(G[it % 6], V, U, O)
    info = eng.info()
    for l, (s, i) in enumerate(zip(specs, info)):
        if s.selector == 0 and l not in (0, 11):
            continue
        lc = list(i["level_count"][:i["iters"]])
        lt = [round(x / 1e-2, 3) for x in i["level_thresh"][:i["iters"]]]
        print(f"it {it:2d} l{l:2d} q{s.quantize} sel{s.selector} flags {i['flags']:#x} cnt {i['count']:7d} "
              f"k {int(s.n*0.001+0.999):6d} iters {i['iters']} lb {i['lb_mask']:#x} stashed {i['stashed']} "
              f"counts {lc} thr/sigma {lt}")
        if s.selector == 1:
            dbg = R.rgc_debug_layer(eng.ctx, eng.ws, l)
            import struct
            f = lambda k: round(struct.unpack("<f", struct.pack("<I", k))[0] / 1e-2, 3)
            print("      ", {k: (f(v) if k in ("thr_key", "stash_key") else v) for k, v in dbg.items()})
