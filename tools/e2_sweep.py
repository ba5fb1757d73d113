"""E2 analog: compression time of one layer of n elements vs n for the
paper's selectors -- trimmed top-k (Alg.2), threshold binary search (Alg.3), sampled threshold
search (interval 5) -- and the paper's comparator, an exact top-k by radix select over the
whole residual (trim_eps = 0.9999: one Alg.2 level near the mean, its survivors overflow the
survivor buffer, so the layer takes the exact radix-select path over V).

Synthetic N(0, 0.01^2) gradients, D = 0.001, m = 0.9, warm residuals (10 calls before timing),
a fresh gradient each call; rgc_compress timed with CUDA events on its stream, median of 5
blocks of 8 calls.  Prints one JSON document (and writes --out).
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1808_04357_b200 import rgc as R  # noqa: E402

VARIANTS = {
    "trimmed": dict(selector=0),
    "threshold_bs": dict(selector=1),
    "sampled_bs": dict(selector=2, sample_interval=5),
    "radix_select": dict(selector=0, trim_eps=0.9999),
}


def time_variant(n, kw, dev, gen, warm=10):
    """warm calls with a fresh gradient each, then 5 timed blocks of 8 calls (fresh
    gradients generated before each block), then 20 calls whose paths are tallied."""
    spec = R.LayerSpec(n=n, density=0.001, momentum=0.9, **kw)
    eng = R.RGC([spec], device=0)
    V = [torch.zeros(n, device=dev)]
    U = [torch.zeros(n, device=dev)]
    g = torch.empty(n, device=dev)
    for i in range(warm):
        torch.randn(n, device=dev, generator=gen, out=g)
        g.mul_(0.01)
        eng.compress([g], V, U)
    torch.cuda.synchronize()
    blocks = []
    G = [torch.empty(n, device=dev) for _ in range(8)]
    for b in range(5):
        for x in G:
            torch.randn(n, device=dev, generator=gen, out=x)
            x.mul_(0.01)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(8):
            eng.compress([G[i]], V, U)
        e1.record()
        torch.cuda.synchronize()
        blocks.append(e0.elapsed_time(e1) / 8)
    paths = {"reuse": 0, "reuse_cap_exact": 0, "search": 0, "cap_exact": 0, "calls": 20}
    counts = []
    for i in range(20):
        torch.randn(n, device=dev, generator=gen, out=g)
        g.mul_(0.01)
        eng.compress([g], V, U)
        f = eng.info()[0]
        counts.append(int(f["count"]))
        if f["flags"] & R.F_SAMPLED_REUSE:
            paths["reuse_cap_exact" if f["flags"] & R.F_CAP_EXACT else "reuse"] += 1
        else:
            paths["cap_exact" if f["flags"] & R.F_CAP_EXACT else "search"] += 1
    info = eng.info()[0]
    eng.close()
    return statistics.median(blocks), info, paths, counts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--sizes", default="65536,262144,1048576,4194304,16777216,67108864,100000000")
    ap.add_argument("--warm", type=int, default=10,
                    help="warm calls before timing (10: drifting residual; ~3000: the residual "
                         "distribution has reached its steady state, every element was sent)")
    ap.add_argument("--variants", default=",".join(VARIANTS))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    rows = []
    for n in [int(x) for x in args.sizes.split(",")]:
        row = {"n": n}
        names = args.variants.split(",")
        for name in names:
            ms, info, paths, counts = time_variant(n, VARIANTS[name], dev, gen, args.warm)
            row[name] = {"ms": ms, "GBps": 4 * n / (ms * 1e-3) / 1e9, "flags": int(info["flags"]),
                         "count": int(info["count"]), "paths": paths,
                         "count_over_k": [c / max(1, -(-n // 1000)) for c in counts]}
        base = row.get("radix_select", row.get("threshold_bs"))["ms"]
        for name in names:
            row[name]["speedup_vs_base"] = base / row[name]["ms"]
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    doc = {"tool": "e2_sweep", "density": 0.001, "momentum": 0.9, "data": "synthetic N(0, 0.01^2)",
           "warm_calls": args.warm, "speedup_base": "radix_select if timed, else threshold_bs",
           "timing": "rgc_compress per call, CUDA events, median of 5 blocks of 8 calls",
           "rows": rows}
    print(json.dumps(doc))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
