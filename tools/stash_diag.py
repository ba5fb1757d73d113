"""Per-layer candidate-stash statistics of the VGG16 bench workload after warm-up: records
K1 stashed, the selected count / survivors they serve, the stash key and the Alg.3 hint and
margin (what K2/K3 read in place of the residual)."""
import os
import struct
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1808_04357_b200 import rgc as R  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
policy = sys.argv[2] if len(sys.argv) > 2 else "hybrid"
dist = sys.argv[3] if len(sys.argv) > 3 else "gaussian"
specs, sizes, kinds = bench.layer_specs(wl, policy, False)
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev)
gen.manual_seed(1)
G = [[bench.device_gradient(n, dist, dev, gen) for n in sizes] for _ in range(6)]
V = [torch.zeros(n, device=dev) for n in sizes]
U = [torch.zeros(n, device=dev) for n in sizes]
O = [torch.empty(n, device=dev) for n in sizes]
eng = R.RGC(specs, device=0)
f = lambda k: struct.unpack("<f", struct.pack("<I", k))[0]  # noqa: E731
tot = 0
iters = int(os.environ.get("ITERS", "40"))
miss = [0] * len(specs)
for it in range(iters):
    eng.step(G[it % 6], V, U, O)
    torch.cuda.synchronize()
    if it < 8:
        continue
    info = eng.info()
    for l, s in enumerate(specs):
        d = R.rgc_debug_layer(eng.ctx, eng.ws, l)
        miss[l] += 0 if d["k2_from_stash"] and d["k3_from_stash"] else 1
        if s.n >= int(os.environ.get("TRACE_N", "4000000")) and it % int(os.environ.get("TRACE_EVERY", "4")) == 0:
            print(f"  it {it:2d} l{l} records {d['stash_records']:8d} need {d['need_count']:8d} "
                  f"count {d['count']:7d} shift {d['stash_shift']} margin {d['bs_margin']} "
                  f"hint {d['bs_hint']} thr {f(d['thr_key']):.4f} key {f(d['stash_key']):.4f} "
                  f"max {f(info[l]['maxkey']):.3f} k2s {d['k2_from_stash']} k3s {d['k3_from_stash']} "
                  f"vp {d['vpass_runs']} full {d['full_runs']}")
print("stash misses per layer over", iters - 8, "steps:", miss)
print("V-pass runs", [R.rgc_debug_layer(eng.ctx, eng.ws, l)["vpass_runs"] for l in range(len(specs))])
print("full-histogram runs", [R.rgc_debug_layer(eng.ctx, eng.ws, l)["full_runs"] for l in range(len(specs))])
info = eng.info()
for l, (s, i) in enumerate(zip(specs, info)):
    d = R.rgc_debug_layer(eng.ctx, eng.ws, l)
    tot += d["stash_records"]
    print(f"l{l:2d} n {s.n:10d} sel {s.selector} count {i['count']:7d} surv {i['survivors']:7d} "
          f"records {d['stash_records']:8d} ({d['stash_records'] / s.n * 100:5.2f}%) "
          f"thr {f(d['thr_key']):.5f} key {f(d['stash_key']):.5f} shift {d['stash_shift']} "
          f"need {d['need_count']} hint {d['bs_hint']} margin {d['bs_margin']} k2s {d['k2_from_stash']} "
          f"k3s {d['k3_from_stash']}")
print(f"total records {tot} = {tot * 8 / 1e6:.1f} MB ({tot / sum(sizes) * 100:.2f}% of {sum(sizes)})")
