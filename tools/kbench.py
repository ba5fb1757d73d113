"""Quick phase timing of the RGC path on one GPU (development tool, not the bench contract)."""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1808_04357_b200 import rgc as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="vgg16")
    ap.add_argument("--policy", default="hybrid")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--dist", default="gaussian")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    sizes, kinds = synth.model_layers(args.model)
    specs = [R.LayerSpec(n=n, density=0.001, momentum=0.9,
                         selector=synth.selector_for(args.model, k, args.policy))
             for n, k in zip(sizes, kinds)]
    eng = R.RGC(specs, device=0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(0)
    G = [torch.randn(n, device=dev, generator=gen) * 0.01 for n in sizes]
    if args.dist == "uniform":
        G = [torch.rand(n, device=dev, generator=gen) for n in sizes]
    V = [torch.zeros(n, device=dev) for n in sizes]
    U = [torch.zeros(n, device=dev) for n in sizes]
    O = [torch.empty(n, device=dev) for n in sizes]
    for _ in range(args.warmup):
        eng.step(G, V, U, O)
    torch.cuda.synchronize()
    R.rgc_profile(eng.ctx, True)
    R.rgc_profile_read(eng.ctx)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.iters):
        eng.step(G, V, U, O)
    e1.record()
    torch.cuda.synchronize()
    ph, n = R.rgc_profile_read(eng.ctx)
    tot = e0.elapsed_time(e1) / args.iters
    N = sum(sizes)
    res = {"model": args.model, "policy": args.policy, "dist": args.dist, "ms_per_iter": tot,
           "phase_ms": {k: v / args.iters for k, v in ph.items()},
           "compress_GBps_grad": 4 * N / (sum(list(ph.values())[:5]) / args.iters * 1e-3) / 1e9,
           "k1_GBps_alg": 20 * N / (ph["accumulate"] / args.iters * 1e-3) / 1e9,
           "k2_GBps_alg": 4 * N / (ph["count_search"] / args.iters * 1e-3) / 1e9,
           "k3_GBps_alg": 4 * N / (ph["compact"] / args.iters * 1e-3) / 1e9,
           "decomp_GBps_alg": 4 * N / (ph["decompress"] / args.iters * 1e-3) / 1e9}
    info = eng.info()
    res["flags"] = [hex(i["flags"]) for i in info]
    res["counts"] = [i["count"] for i in info]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
