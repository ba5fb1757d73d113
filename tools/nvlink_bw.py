"""NVLink peer copy bandwidth between the visible GPUs (one process; development tool).

Measures, with CUDA events on the source device's stream, a device-to-device peer copy
(`dst.copy_(src)` across devices = cudaMemcpyPeerAsync over NVLink / NVSwitch) of 1 MB ... 1 GB
from GPU 0 to every other GPU, one direction and both directions at once, best of 10 per
size.  The largest-size unidirectional figure is the peak bench.py divides the exchange's
GB/s by (`profiles/r02/nvlink_peak.json`; the guide's reference is 770 GB/s per direction).

    python tools/nvlink_bw.py --out profiles/r02/nvlink_peak.json
"""
import argparse
import json
import time

import torch


def bench_copy(src, dst, reps=10):
    s = torch.cuda.current_stream(src.device)
    best = 1e30
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(src.device)
    torch.cuda.synchronize(dst.device)
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(src.device):
            e0.record(s)
            dst.copy_(src, non_blocking=True)
            e1.record(s)
        e1.synchronize()
        torch.cuda.synchronize(dst.device)
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n = torch.cuda.device_count()
    res = {"tool": "nvlink_bw", "gpus": n, "gpu_name": torch.cuda.get_device_name(0),
           "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "method": "dst.copy_(src) across devices (cudaMemcpyPeerAsync), CUDA events on the "
                     "source stream, best of 10", "pairs": []}
    if n < 2:
        res["error"] = "needs 2 GPUs"
        print(json.dumps(res))
        return
    for i in range(n):
        for j in range(n):
            if i != j:
                try:
                    torch.cuda.set_device(i)
                    ok = torch.cuda.can_device_access_peer(i, j)
                except Exception:
                    ok = False
                res.setdefault("peer_access", {})[f"{i}->{j}"] = bool(ok)
    sizes = [1 << 20, 8 << 20, 64 << 20, 256 << 20, 1 << 30]
    for j in range(1, n):
        row = {"src": 0, "dst": j, "uni_GBps": {}, "bidir_GBps_per_direction": {}}
        for b in sizes:
            a = torch.empty(b, dtype=torch.uint8, device="cuda:0")
            c = torch.empty(b, dtype=torch.uint8, device=f"cuda:{j}")
            ms = bench_copy(a, c)
            row["uni_GBps"][str(b)] = b / ms / 1e6
            # both directions at once: two copies on the two devices' streams
            a2 = torch.empty(b, dtype=torch.uint8, device=f"cuda:{j}")
            c2 = torch.empty(b, dtype=torch.uint8, device="cuda:0")
            best = 1e30
            for _ in range(5):
                torch.cuda.synchronize(0)
                torch.cuda.synchronize(j)
                t0 = time.perf_counter()
                with torch.cuda.device(0):
                    c.copy_(a, non_blocking=True)
                with torch.cuda.device(j):
                    c2.copy_(a2, non_blocking=True)
                torch.cuda.synchronize(0)
                torch.cuda.synchronize(j)
                best = min(best, time.perf_counter() - t0)
            row["bidir_GBps_per_direction"][str(b)] = b / best / 1e9
            del a, c, a2, c2
        res["pairs"].append(row)
    big = str(sizes[-1])
    res["peak_uni_GBps"] = max(r["uni_GBps"][big] for r in res["pairs"])
    res["peak_bidir_GBps_per_direction"] = max(r["bidir_GBps_per_direction"][big] for r in res["pairs"])
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
