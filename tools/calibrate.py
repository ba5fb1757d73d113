#!/usr/bin/env python
"""NEXT-4: calibrate the paper's cost model on this box and put the measured
RGC synchronisation next to it and next to the dense NCCL Allreduce it replaces.

  python tools/calibrate.py                                  # 1 GPU: gamma_1, T_select
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      --master-port P tools/calibrate.py                     # + alpha, beta, gamma_2

Measured (CUDA events, median of repeats, max over ranks):
  * NCCL Allgather of b bytes per rank           -> alpha, beta      (Eq. (1) transfer)
  * NCCL Allreduce of b bytes (fp32 sum)         -> alpha_d, gamma_2 (Eq. (2), beta shared)
  * rgc_decompress of p' messages of a layer     -> fixed + p' gamma_1
  * the VGG16 RGC step (compress / sync / decompress phases) -> T_select and the sync
  * one dense NCCL Allreduce of all VGG16 gradients (the paper's SGD comparator)
and Eq. (1) / Eq. (2) evaluated with the fitted parameters for the VGG16 step.
Prints one JSON line (rank 0); --out writes it to a file too.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_1808_04357_b200 import costmodel as CM  # noqa: E402
from paper_1808_04357_b200 import rgc as R  # noqa: E402


def timed(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    s = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    return statistics.median(ts)


def max_over_ranks(x, world, dev):
    t = torch.tensor([x], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--workload", default="vgg16")
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    with bench.stdout_to_stderr():
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
    res = {"tool": "calibrate", "n_gpus": world, "workload": args.workload,
           "units": "seconds, bytes", "model": "Eq. (1) / Eq. (2) of P:360-366"}

    # ---- collectives: alpha, beta (Allgather), alpha_d, gamma_2 (Allreduce)
    if world > 1:
        ag = []
        for b in [1 << e for e in range(12, 25, 2)]:           # 4 KB .. 16 MB per rank
            x = torch.zeros(b, dtype=torch.uint8, device=dev)
            y = torch.zeros(b * world, dtype=torch.uint8, device=dev)
            t = timed(lambda: dist.all_gather_into_tensor(y, x), 20)
            ag.append((world, b, max_over_ranks(t, world, dev)))
        ar = []
        for b in [1 << e for e in range(16, 30, 2)]:           # 64 KB .. 256 MB
            x = torch.ones(b // 4, dtype=torch.float32, device=dev)
            t = timed(lambda: dist.all_reduce(x), 10)
            ar.append((world, b, max_over_ranks(t, world, dev)))
        alpha, beta = CM.fit_allgather(ag)
        alpha_d, _, g2 = CM.fit_allreduce(ar, beta=beta)
        _, beta_eff, _ = CM.fit_allreduce(ar)
        res["allgather_samples"] = ag
        res["allreduce_samples"] = ar
        res["fit"] = {"alpha": alpha, "beta": beta, "alpha_dense": alpha_d,
                      "gamma2_per_byte": g2, "beta_dense_eff": beta_eff,
                      "allgather_GBps": 1e-9 / beta if beta > 0 else None,
                      "allreduce_busbw_GBps": 1e-9 / beta_eff if beta_eff > 0 else None}
    else:
        alpha = beta = alpha_d = g2 = 0.0

    # ---- gamma_1: decompress p' collected messages of the largest layer (simulated ranks)
    specs, sizes, _ = bench.layer_specs(args.workload, "hybrid")
    big = max(range(len(sizes)), key=lambda i: sizes[i])
    sp = [specs[big]]
    M = sizes[big]
    one = R.RGC(sp, nranks=1, device=local)
    V = [torch.zeros(M, device=dev)]
    U = [torch.zeros(M, device=dev)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(77 + rank)
    blocks = []
    for i in range(16):
        g = [torch.randn(M, device=dev, generator=gen) * 0.01]
        one.compress(g, V, U)
        blocks.append(one.msg.clone())
    one.close()
    dec_samples = []
    out = [torch.empty(M, device=dev)]
    for pp in (1, 2, 4, 8, 16):
        eng = R.RGC(sp, nranks=pp, device=local) if pp > 1 else None
        if eng is None:
            eng = R.RGC(sp, nranks=1, device=local)
            eng.gathered.copy_(blocks[0])
        else:
            eng.gathered.copy_(torch.cat(blocks[:pp]))
        eng.prefill = False
        t = timed(lambda: eng.decompress(out), 10)
        dec_samples.append((pp, t))
        eng.close()
    fixed, gamma1 = CM.fit_decompress(dec_samples)
    res["decompress_samples"] = {"layer_elements": M, "density": specs[big].density,
                                 "samples": dec_samples, "fixed": fixed, "gamma1": gamma1}

    # ---- the RGC step of the workload (P2P exchange for N > 1) and the dense comparator
    mode = R.RGC_SYNC_P2P if world > 1 else R.RGC_SYNC_FIXED
    with bench.stdout_to_stderr():
        uid = None
        if world > 1:
            obj = [R.rgc_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        eng = R.RGC(specs, rank=rank, nranks=world, device=local, uid=uid, sync_mode=mode)
    G = [[torch.randn(n, device=dev, generator=gen) * 0.01 for n in sizes] for _ in range(4)]
    V = [torch.zeros(n, device=dev) for n in sizes]
    U = [torch.zeros(n, device=dev) for n in sizes]
    O = [torch.empty(n, device=dev) for n in sizes]
    for i in range(8):
        eng.step(G[i % 4], V, U, O)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    R.rgc_profile(eng.ctx, True)
    R.rgc_profile_read(eng.ctx)
    step_t = timed(lambda: eng.step(G[0], V, U, O), args.steps, warm=0)
    ph, _ = R.rgc_profile_read(eng.ctx)
    R.rgc_profile(eng.ctx, False)
    n_prof = args.steps
    ph = {k: max_over_ranks(v * 1e-3 / n_prof, world, dev) for k, v in ph.items()}
    step_t = max_over_ranks(step_t, world, dev)
    counts = [int(i["count"]) for i in eng.info()]
    H = eng.header_words()
    msg_bytes = 4 * H + 8 * sum(counts)
    eng.close()
    N = sum(sizes)
    dense_t = None
    if world > 1:
        flat = torch.ones(N, dtype=torch.float32, device=dev)
        dense_t = max_over_ranks(timed(lambda: dist.all_reduce(flat), 5), world, dev)
        del flat
    t_select = sum(ph[k] for k in R.PHASES[:5])
    c = CM.CostParams(alpha=alpha, beta=beta, gamma1=gamma1, gamma2=g2 * 4 * N, t_select=t_select)
    Deff = sum(counts) / N
    # Eq. (1) for the step's one bucketed message (bytes per rank = the used message bytes)
    pred_sparse = (c.t_select + CM.lg(world) * c.alpha + (world - 1) * msg_bytes * c.beta
                   + world * gamma1 * (N / M) + fixed * (N / M))
    pred_dense = CM.t_dense(c, world, N, "byte") if world > 1 else None
    res["step"] = {"measured_ms": step_t * 1e3, "phases_ms": {k: v * 1e3 for k, v in ph.items()},
                   "t_select_ms": t_select * 1e3, "message_bytes_per_rank": msg_bytes,
                   "effective_density": Deff,
                   "eq1_predicted_ms": pred_sparse * 1e3,
                   "eq1_note": "T_select measured; transfer from the Allgather fit; p gamma_1 and "
                               "the fixed decompress cost scaled from the largest layer by elements"}
    res["dense_allreduce"] = {"measured_ms": dense_t * 1e3 if dense_t else None,
                              "eq2_predicted_ms": pred_dense * 1e3 if pred_dense else None,
                              "bytes": 4 * N,
                              "rgc_speedup": (dense_t / step_t) if dense_t else None}
    if world > 1:
        res["crossover_density"] = CM.crossover_density(
            CM.CostParams(alpha=alpha, beta=beta, gamma1=gamma1, gamma2=g2 * 4 * N,
                          t_select=t_select), world, N, "byte")
        res["bandwidth_coefficient"] = CM.bandwidth_coefficient(world, Deff)
    if rank == 0:
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line + "\n")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
