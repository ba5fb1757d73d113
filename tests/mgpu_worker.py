"""Multi-GPU parity worker (launched by tests/test_multigpu.py under torchrun).

Every rank compresses its own seeded gradients through the C ABI, rgc_sync
exchanges the messages (NCCL allgather, NCCL sizes-first, RGC_SYNC_P2P where
every rank pushes its block into the peers over NVLink, or RGC_SYNC_PULL where
rgc_decompress reads every peer's block in place over NVLink), and rgc_decompress
produces the dense averaged gradient.  Checks:
  AGREEMENT: every rank holds byte-identical gathered buffers;
  parity: rank 0 re-runs all p ranks in the CPU oracle from the same seeds and
  compares residuals, messages and the decompressed average bit-exactly;
  PULL pipelined: several iterations enqueued back to back with no host
  synchronisation and rank 0 delayed before each decompression, so a producer's
  next compress must wait for the slow reader (the write-after-read guard).
"""
import hashlib
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle as O  # noqa: E402
import synth  # noqa: E402
from harness import bits, compare_info  # noqa: E402
from paper_1808_04357_b200 import rgc as R  # noqa: E402


def pull_pipelined(specs, dists, rank, world, local, dev, iters=4):
    """RGC_SYNC_PULL with no host synchronisation between iterations: rank 0 spins
    ~50 ms on its stream before every decompression, so the other ranks reach their
    next compress while rank 0 still has to read their blocks; K1's wait for
    "consumed" must keep them from rewriting the blocks early.  Outputs and
    residuals of every iteration are cloned on the stream and compared with the
    oracle at the end."""
    failures = []
    uid = [R.rgc_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng = R.RGC(specs, rank=rank, nranks=world, device=local, uid=uid[0],
                sync_mode=R.RGC_SYNC_PULL)
    V = [torch.zeros(s.n, device=dev) for s in specs]
    U = [torch.zeros(s.n, device=dev) if s.momentum else None for s in specs]
    out = [torch.empty(s.n, device=dev) for s in specs]
    grads = [[torch.from_numpy(synth.gradient(s.n, dists[l], seed=11, rank=rank, layer=l, it=it)).to(dev)
              for l, s in enumerate(specs)] for it in range(iters)]
    torch.cuda.synchronize()
    dist.barrier()
    outs_hist, v_hist = [], []
    for it in range(iters):
        eng.compress(grads[it], V, U)
        eng.sync()
        if rank == 0:
            torch.cuda._sleep(100_000_000)   # ~50 ms at ~2 GHz: rank 0 reads late
        eng.decompress(out)
        outs_hist.append([o.clone() for o in out])
        v_hist.append([v.clone() for v in V])
    torch.cuda.synchronize()
    outs_all = [None] * world
    dist.all_gather_object(outs_all, [[o.cpu().numpy().view(np.uint32).tobytes() for o in oo]
                                      for oo in outs_hist])
    vs_all = [None] * world
    dist.all_gather_object(vs_all, [[v.cpu().numpy().view(np.uint32).tobytes() for v in vv]
                                    for vv in v_hist])
    if rank == 0:
        Vo = [[np.zeros(s.n, np.float32) for s in specs] for _ in range(world)]
        Uo = [[np.zeros(s.n, np.float32) if s.momentum else None for s in specs] for _ in range(world)]
        Ao = [[O.AsqState() if s.quantize else None for s in specs] for _ in range(world)]
        for it in range(iters):
            om = [[None] * len(specs) for _ in range(world)]
            for r in range(world):
                for l, s in enumerate(specs):
                    gr = synth.gradient(s.n, dists[l], seed=11, rank=r, layer=l, it=it)
                    idx, val, oi = O.compress_layer(gr, Uo[r][l], Vo[r][l], s.momentum, s.density,
                                                    s.selector, s.bs_branch, asq=Ao[r][l])
                    if s.quantize:
                        val = np.full(len(idx), oi["qmean"], np.float32)
                    om[r][l] = (idx, val)
                    if vs_all[r][it][l] != bits(Vo[r][l]).tobytes():
                        failures.append(f"PULL pipelined it {it} r{r} l{l}: residual differs")
            for l, s in enumerate(specs):
                want = bits(O.decompress(s.n, [om[r][l] for r in range(world)])).tobytes()
                for r in range(world):
                    if outs_all[r][it][l] != want:
                        failures.append(f"PULL pipelined it {it} r{r} l{l}: decompress differs")
    eng.close()
    return failures


def status_scenarios(rank, world, local, dev):
    """rgc_status across ranks (include/rgc.h): (1) one rank's non-finite residual reaches
    every rank's context status through the exchanged status words (P2P push); (2) a wait
    for a peer that stays away longer than RGC_P2P_TIMEOUT_S becomes a hard RGC_ESTATE on the
    waiting rank, and that context refuses further work."""
    import time
    failures = []
    specs = [R.LayerSpec(n=100_000, density=0.001, momentum=0.9, selector=0),
             R.LayerSpec(n=50_000, density=0.001, momentum=0.9, selector=1)]
    V = [torch.zeros(s.n, device=dev) for s in specs]
    U = [torch.zeros(s.n, device=dev) for s in specs]
    out = [torch.empty(s.n, device=dev) for s in specs]
    g = [torch.from_numpy(synth.gradient(s.n, "gaussian", seed=5, rank=rank, layer=l)).to(dev)
         for l, s in enumerate(specs)]
    # (1) non-finite on rank world-1 only
    uid = [R.rgc_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng = R.RGC(specs, rank=rank, nranks=world, device=local, uid=uid[0], sync_mode=R.RGC_SYNC_P2P)
    eng.step(g, V, U, out)
    rc, w = eng.status()
    if rc != R.RGC_OK:
        failures.append(f"status: clean step reported {rc} {w}")
    if rank == world - 1:
        g[1][777] = float("inf")
    try:
        eng.step(g, V, U, out)   # its own poll may already see the error (a fast step)
    except R.RgcError as e:
        if e.code != R.RGC_ENONFINITE:
            failures.append(f"status: non-finite step raised {e.code}")
    rc, w = eng.status()
    if rc != R.RGC_ENONFINITE or not (w[0] & R.F_NONFINITE):
        failures.append(f"status: rank {rank} did not see rank {world - 1}'s non-finite residual ({rc}, {w})")
    torch.cuda.synchronize()
    dist.barrier()
    eng.close()
    # (2) timeout: rank 1 arrives 4 s late; rank 0 waits at most 1 s
    os.environ["RGC_P2P_TIMEOUT_S"] = "1"
    uid = [R.rgc_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    eng = R.RGC(specs, rank=rank, nranks=world, device=local, uid=uid[0], sync_mode=R.RGC_SYNC_P2P)
    del os.environ["RGC_P2P_TIMEOUT_S"]
    g[1].zero_()
    for v, u in zip(V, U):   # scenario (1) left Inf in rank world-1's residual and momentum
        v.zero_()
        u.zero_()
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 1:
        time.sleep(4.0)
    try:
        eng.step(g, V, U, out)
    except R.RgcError as e:
        if not (rank == 0 and e.code == R.RGC_ESTATE):
            failures.append(f"status: late-peer step raised {e.code} on rank {rank}")
    rc, w = eng.status()
    if rank == 0:
        if rc != R.RGC_ESTATE or not (w[0] & R.STAT_TIMEOUT) or not (w[1] & 2):
            failures.append(f"status: rank 0's timed-out wait for rank 1 gave ({rc}, {w})")
        try:
            eng.compress(g, V, U)
            failures.append("status: a timed-out context accepted more work")
        except R.RgcError as e:
            if e.code != R.RGC_ESTATE:
                failures.append(f"status: timed-out context refused work with {e.code}")
    torch.cuda.synchronize()
    dist.barrier()
    eng.close()
    return failures


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import datetime
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=240))
    specs = [R.LayerSpec(n=1_000_000, density=0.001, momentum=0.9, selector=0),
             R.LayerSpec(n=262_147, density=0.001, momentum=0.9, selector=1),
             R.LayerSpec(n=4097, density=0.01, momentum=0.0, selector=1, bs_branch=1),
             R.LayerSpec(n=150_001, density=0.001, momentum=0.9, selector=0),
             R.LayerSpec(n=300_007, density=0.001, momentum=0.9, selector=0, quantize=1),
             R.LayerSpec(n=200_003, density=0.002, momentum=0.9, selector=1, quantize=1)]
    dists = ["gaussian", "t3", "gaussian", "laplace", "gaussian", "t3"]
    failures = []
    for mode in (R.RGC_SYNC_FIXED, R.RGC_SYNC_SIZES_FIRST, R.RGC_SYNC_P2P, R.RGC_SYNC_PULL):
        print(f"rank {rank}: mode {mode}", file=sys.stderr, flush=True)
        uid = [R.rgc_get_unique_id() if rank == 0 else None]   # one id per communicator
        dist.broadcast_object_list(uid, src=0)
        eng = R.RGC(specs, rank=rank, nranks=world, device=local, uid=uid[0], sync_mode=mode,
                    p2p_inspect=True)
        V = [torch.zeros(s.n, device=dev) for s in specs]
        U = [torch.zeros(s.n, device=dev) if s.momentum else None for s in specs]
        out = [torch.empty(s.n, device=dev) for s in specs]
        if rank == 0:
            Vo = [[np.zeros(s.n, np.float32) for s in specs] for _ in range(world)]
            Uo = [[np.zeros(s.n, np.float32) if s.momentum else None for s in specs]
                  for _ in range(world)]
            Ao = [[O.AsqState() if s.quantize else None for s in specs] for _ in range(world)]
        for it in range(3):
            g = [synth.gradient(s.n, dists[l], seed=7, rank=rank, layer=l, it=it)
                 for l, s in enumerate(specs)]
            eng.compress([torch.from_numpy(x).to(dev) for x in g], V, U)
            counts = np.zeros(world * len(specs), np.uint32) if mode == R.RGC_SYNC_SIZES_FIRST else None
            eng.sync(counts_host=counts)
            eng.decompress(out)
            torch.cuda.synchronize()
            # AGREEMENT: digest of the gathered blocks (the used part of each block)
            msgs = eng.messages()
            h = hashlib.sha256()
            for r in range(world):
                for l in range(len(specs)):
                    h.update(msgs[r][l][0].tobytes())
                    h.update(msgs[r][l][1].tobytes())
            digests = [None] * world
            dist.all_gather_object(digests, h.hexdigest())
            if len(set(digests)) != 1:
                failures.append(f"mode {mode} it {it}: gathered buffers differ across ranks")
            outs = [o.cpu().numpy() for o in out]
            outs_all = [None] * world
            dist.all_gather_object(outs_all, [o.view(np.uint32).tobytes() for o in outs])
            Vs_all = [None] * world
            dist.all_gather_object(Vs_all, [v.cpu().numpy().view(np.uint32).tobytes() for v in V])
            infos = [None] * world
            dist.all_gather_object(infos, eng.info())
            if rank == 0:
                for r in range(1, world):
                    if outs_all[r] != outs_all[0]:
                        failures.append(f"mode {mode} it {it}: decompressed outputs differ r{r}")
                om = [[None] * len(specs) for _ in range(world)]
                for r in range(world):
                    for l, s in enumerate(specs):
                        gr = synth.gradient(s.n, dists[l], seed=7, rank=r, layer=l, it=it)
                        idx, val, oi = O.compress_layer(gr, Uo[r][l], Vo[r][l], s.momentum,
                                                        s.density, s.selector, s.bs_branch,
                                                        asq=Ao[r][l])
                        if s.quantize:   # ASQ: the message carries the indices and one mean
                            val = np.full(len(idx), oi["qmean"], np.float32)
                        om[r][l] = (idx, val)
                        try:
                            compare_info(infos[r][l], oi, s, f"mode {mode} it {it} r{r} l{l}")
                        except AssertionError as e:
                            failures.append(str(e))
                        gi, gv = msgs[r][l]
                        if not (np.array_equal(gi, idx) and np.array_equal(bits(gv), bits(val))):
                            failures.append(f"mode {mode} it {it} r{r} l{l}: message differs")
                        if np.frombuffer(Vs_all[r][l], np.uint32).tobytes() != bits(Vo[r][l]).tobytes():
                            failures.append(f"mode {mode} it {it} r{r} l{l}: residual differs")
                        if counts is not None and counts[r * len(specs) + l] != len(idx):
                            failures.append(f"mode {mode} it {it} r{r} l{l}: counts_host differs")
                for l, s in enumerate(specs):
                    want = O.decompress(s.n, [om[r][l] for r in range(world)])
                    if np.frombuffer(outs_all[0][l], np.uint32).tobytes() != bits(want).tobytes():
                        failures.append(f"mode {mode} it {it} l{l}: decompress differs from oracle")
        eng.close()
    print(f"rank {rank}: modes done", file=sys.stderr, flush=True)
    failures += pull_pipelined(specs, dists, rank, world, local, dev)
    print(f"rank {rank}: pull pipelined done", file=sys.stderr, flush=True)
    failures += status_scenarios(rank, world, local, dev)
    print(f"rank {rank}: status scenarios done", file=sys.stderr, flush=True)
    res = [None] * world
    dist.all_gather_object(res, failures)
    dist.destroy_process_group()
    if rank == 0:
        allf = [f for r in res for f in r]
        print("MGPU_RESULT", "OK" if not allf else "FAIL", len(allf))
        for f in allf[:20]:
            print("  ", f)
        sys.exit(0 if not allf else 1)


if __name__ == "__main__":
    main()
