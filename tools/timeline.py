"""Per-kernel timeline of a warm step (development tool): every kernel's earliest CTA start
(after its programmatic-dependent-launch wait) and latest CTA exit, relative to K1's start,
median over steps -- the chain as it runs, with the zero fill beside it (ncu serialises).

    python tools/timeline.py [--workload vgg16] [--policy hybrid] [--steps 10]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RGC_TIMELINE"] = "1"
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1808_04357_b200 import rgc as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="vgg16")
    ap.add_argument("--policy", default="hybrid")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=10)
    args = ap.parse_args()
    specs, sizes, _ = bench.layer_specs(args.workload, args.policy)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    G = [[torch.randn(n, device=dev, generator=gen) * 0.01 for n in sizes] for _ in range(4)]
    V = [torch.zeros(n, device=dev) for n in sizes]
    U = [torch.zeros(n, device=dev) for n in sizes]
    O = [torch.empty(n, device=dev) for n in sizes]
    eng = R.RGC(specs, device=0)
    for i in range(args.warmup):
        eng.step(G[i % 4], V, U, O)
    torch.cuda.synchronize()
    rows = {}
    step_us = []
    for i in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.step(G[i % 4], V, U, O)
        e1.record()
        torch.cuda.synchronize()
        step_us.append(e0.elapsed_time(e1) * 1e3)
        for k, (a, b) in R.rgc_debug_timeline(eng.ctx).items():
            rows.setdefault(k, []).append((a, b))
    eng.close()
    res = {k: {"start_us": statistics.median(x[0] for x in v),
               "end_us": statistics.median(x[1] for x in v)} for k, v in rows.items()}
    order = sorted(res, key=lambda k: res[k]["start_us"])
    print(json.dumps({"workload": args.workload, "policy": args.policy,
                      "step_us_median": statistics.median(step_us),
                      "timeline": {k: res[k] for k in order}}, indent=1))


if __name__ == "__main__":
    main()
