#!/usr/bin/env python
"""Benchmark of the RedSync RGC synchronisation hot path on B200 (bench contract).

One step = one pass of the whole hot path over one iteration's gradients of the
workload: rgc_compress (all compressed layers: accumulate + momentum correction,
selection, compaction, residual masking) -> rgc_sync (allgather over NCCL/NVLink)
-> rgc_decompress (rank-ordered dense averaged gradient).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload vgg16]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference      # the CPU oracle as the reference arm

Metric (BASELINE.json): "RGC sync ms/iter and compress GB/s (HBM roofline %) at
D=0.001, 1/2/4/8 B200".  value = ms per iteration (max over ranks, CUDA events,
lower is better); compress GB/s and the HBM roofline of the dominant kernel (K1)
are reported beside it.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RGC sync ms/iter and compress GB/s (HBM roofline %) at D=0.001, 1/2/4/8 B200"
UNIT = "ms/iter"
DENSITY = 0.001
MOMENTUM = 0.9
CONFIG_NOTES = {
    "vgg16": "BASELINE configs[2]: VGG16 ImageNet per-layer gradients (15 compressed tensors, 102.8M-element fc6)",
    "resnet50": "BASELINE configs[1]: ResNet-50 per-layer gradients (45 compressed tensors)",
    "alexnet": "BASELINE configs[3]: AlexNet (7 compressed tensors)",
    "lstm_ptb": "BASELINE configs[4]: 2-layer 1500-hidden LSTM, PTB vocabulary",
    "lstm_wiki2": "BASELINE configs[4]: 2-layer 1500-hidden LSTM, Wiki2 vocabulary",
    "m1": "single 1e8-element gradient (north_star 100M-element kernel target)",
    "c1": "BASELINE configs[0]: single 1M-element gradient",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--pool", type=int, default=0,
                    help="number of distinct gradient sets (default: warmup+steps, <= 64)")
    ap.add_argument("--pool-gb", type=float, default=60.0)
    ap.add_argument("--impl", default="rgc", choices=["rgc", "reference"])
    ap.add_argument("--workload", default="vgg16")
    ap.add_argument("--policy", default="hybrid", choices=["hybrid", "trimmed", "bs"])
    ap.add_argument("--asq", action="store_true",
                    help="Alternating Signs Quantization (P:274-294) on all but the output layer")
    ap.add_argument("--dist", default="gaussian",
                    help="synthetic gradient distribution: gaussian | t3 | laplace | cauchy | uniform")
    ap.add_argument("--sync-mode", default="auto", choices=["auto", "fixed", "sizes_first", "p2p", "pull"],
                    help="auto: p2p (NVLink push, one kernel) for N > 1, fixed for N = 1")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--unordered", action="store_true",
                    help="the unordered atomic decompression (R14: 1e-6 relative) instead of the "
                         "bit-exact rank-ordered one")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step per gradient set in a CUDA graph and replay it")
    ap.add_argument("--buckets", type=int, default=1, choices=[1, 2],
                    help="2: the largest layer in its own RGC context on a second stream, the "
                         "other layers' selection overlapping its accumulate pass (NEXT-3 "
                         "bucketing; one message per bucket)")
    ap.add_argument("--k1-occ-big", type=int, default=2,
                    help="--buckets 2: K1 CTAs per SM of the big bucket (room for the other "
                         "bucket's selection kernels)")
    ap.add_argument("--no-phase-events", action="store_true",
                    help="time the step without per-phase events (phases from a separate loop)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def nvlink_peak():
    """Per-direction NVLink peer-copy bandwidth measured on this pool by tools/nvlink_bw.py
    (profiles/r02/nvlink_peak.json), else the B200_PROFILING.md reference (770 GB/s)."""
    p = os.path.join(ROOT, "profiles", "r02", "nvlink_peak.json")
    try:
        d = json.load(open(p))
        return float(d["peak_uni_GBps"]), "measured (profiles/r02/nvlink_peak.json, peer copy)"
    except Exception:
        return 770.0, "reference (B200_PROFILING.md: peer copy 770 GB/s per direction)"


def ncu_traffic(kernel="k1_accumulate"):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        return d["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.t0 = self.t1 = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}", "--format=csv,noheader",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def start(self):
        self.t0 = time.time()

    def stop(self):
        self.t1 = time.time()

    def result(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = []
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = time.mktime(time.strptime(f[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                ts += float("0." + f[0].split(".")[1]) if "." in f[0] else 0.0
                rows.append((ts, float(f[2].split()[0]), float(f[3].split()[0]), f[6:10]))
            except Exception:
                continue
        inside = [r for r in rows if self.t0 - 0.2 <= r[0] <= self.t1 + 0.2] or rows[-3:]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[1] for r in inside),
                "sm_max_mhz": max(r[2] for r in inside), "reasons": reasons,
                "samples": len(inside)}


DIST_TXT = {"gaussian": "N(0, 0.01^2)", "t3": "Student-t(3) x 0.01", "laplace": "Laplace(0.01)",
            "cauchy": "Cauchy x 0.01", "uniform": "U(0,1)"}


def device_gradient(n, dist, dev, gen, scale=0.01):
    """Seeded synthetic gradient generated on the device (input plumbing, not the path):
    the distributions of synth.gradient (SURVEY 8(d) recipe) -- gaussian N(0, scale^2),
    heavy-tailed Student-t nu=3 x scale (C4), laplace, cauchy, Fig. 3's standard uniform."""
    import torch
    if dist == "gaussian":
        return torch.randn(n, device=dev, generator=gen) * scale
    if dist == "t3":
        z = torch.randn(n, device=dev, generator=gen)
        c = torch.randn(n, 3, device=dev, generator=gen).pow_(2).sum(1)
        return (z / torch.sqrt(c / 3.0)) * scale
    if dist == "laplace":
        u = torch.rand(n, device=dev, generator=gen) - 0.5
        return -torch.sign(u) * torch.log1p(-2 * u.abs()) * scale
    if dist == "cauchy":
        u = torch.rand(n, device=dev, generator=gen)
        return torch.tan(math.pi * (u - 0.5)) * scale
    if dist == "uniform":
        return torch.rand(n, device=dev, generator=gen)
    raise SystemExit(f"--dist {dist}: one of gaussian, t3, laplace, cauchy, uniform")


def layer_specs(workload, policy, asq=False):
    """asq: ASQ on every compressed layer but the output layer, which the
    paper leaves unquantized ("We also do not quantify the output layer")."""
    import synth
    from paper_1808_04357_b200 import rgc as R
    sizes, kinds = synth.model_layers(workload)
    L = len(sizes)
    return [R.LayerSpec(n=n, density=DENSITY, momentum=MOMENTUM,
                        selector=synth.selector_for(workload, k, policy),
                        quantize=1 if asq and l < L - 1 else 0)
            for l, (n, k) in enumerate(zip(sizes, kinds))], sizes, kinds


# --------------------------------------------------------------------- CPU arm
ORACLE_S_PER_ELEMENT = 1.25e-8   # oracle compress+decompress, ~1.7 s per VGG16 iteration (sizing only)


def host_cpu():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


class OracleRunner:
    """The CPU oracle (single-threaded C) over a proportional sample of the workload: layer l
    contributes its first max(1, round(frac * n_l)) elements as a layer of that size (k scales
    with it), so every layer and both selectors are in the sample in proportion.  V, u and the
    ASQ phase persist across steps, so after the warm-up steps the oracle works on warm
    residuals like the GPU does.  One step = compress every layer (rank 0) + decompress (p = 1);
    only the oracle calls are timed (not the gradient generation)."""

    def __init__(self, sizes, sels, quant, frac, seed=0):
        import numpy as np

        import oracle as O
        self.O, self.np = O, np
        self.frac = frac
        self.n = [max(1, int(round(frac * x))) for x in sizes]
        self.sels = sels
        self.V = [np.zeros(n, np.float32) for n in self.n]
        self.U = [np.zeros(n, np.float32) for n in self.n]
        self.asq = [O.AsqState() if quant is not None and quant[l] else None
                    for l in range(len(sizes))]
        self.seed = seed
        self.it = 0

    def step(self):
        import synth
        O, np = self.O, self.np
        tot = 0.0
        for l, (n, sel) in enumerate(zip(self.n, self.sels)):
            g = synth.gradient(n, "gaussian", seed=self.seed, rank=0, layer=l, it=self.it)
            t0 = time.perf_counter()
            idx, val, info = O.compress_layer(g, self.U[l], self.V[l], MOMENTUM, DENSITY, sel,
                                              asq=self.asq[l])
            if self.asq[l] is not None:
                val = np.full(len(idx), info["qmean"], np.float32)
            O.decompress(n, [(idx, val)])
            tot += time.perf_counter() - t0
        self.it += 1
        return tot

    def elements(self):
        return sum(self.n)


class pinned_core:
    """Run the block on one host core (sched_setaffinity), restoring the mask afterwards."""

    def __init__(self):
        self.saved = None
        self.core = None

    def __enter__(self):
        try:
            self.saved = os.sched_getaffinity(0)
            self.core = max(self.saved)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.saved = None
        return self

    def __exit__(self, *exc):
        if self.saved is not None:
            os.sched_setaffinity(0, self.saved)
        return False


def cpu_baseline(sizes, sels, quant=None, frac=0.2, warm=8, steps=8):
    """cpu_baseline of the GPU arm's line (rank 0, N = 1): the oracle as it stands on one
    pinned host core, warm like the GPU (warm steps first), over a proportional sample."""
    run = OracleRunner(sizes, sels, quant, frac, seed=3)
    with pinned_core() as pc:
        for _ in range(warm):
            run.step()
        secs = sum(run.step() for _ in range(steps))
    full = sum(sizes)
    ms_iter = secs * 1e3 / steps * full / run.elements()
    d = {"value": ms_iter, "unit": UNIT, "cores": 1, "kind": "oracle",
         "sample": f"oracle (single-threaded C, -O2) compress+decompress of every layer's leading "
                   f"{frac:.0%} (proportional, {run.elements()} of {full} elements), {warm} warm "
                   f"steps then {steps} timed steps with the residual state carried, scaled to "
                   f"the full iteration ({secs:.2f} s timed)",
         "pinned_core": pc.core}
    d.update(host_cpu())
    return d


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    specs, sizes, kinds = layer_specs(args.workload, args.policy, args.asq)
    sels = [s.selector for s in specs]
    quant = [s.quantize for s in specs]
    full = sum(sizes)
    # every step a proportional sample of every layer, sized so that the whole
    # --steps/--warmup run stays within ~90 s of oracle work
    nsteps = max(1, args.steps + args.warmup)
    frac = min(1.0, max(1e-3, 90.0 / (nsteps * full * ORACLE_S_PER_ELEMENT)))
    run = OracleRunner(sizes, sels, quant, frac, seed=1)
    with pinned_core() as pc:
        for _ in range(args.warmup):
            run.step()
        tot = sum(run.step() for _ in range(args.steps))
    ms_iter = tot * 1e3 / max(1, args.steps) * full / run.elements()
    cb = {"value": ms_iter, "unit": UNIT, "cores": 1, "kind": "oracle", "pinned_core": pc.core,
          "sample": f"every layer's leading {frac:.1%} (proportional: {run.elements()} of {full} "
                    f"elements per step), {args.warmup} warm steps then {args.steps} timed steps "
                    f"with the residual state carried, scaled to the full iteration"}
    cb.update(host_cpu())
    line = {"impl": "reference", "metric": METRIC, "value": ms_iter, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot * 1e3 / max(1, args.steps), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "note": CONFIG_NOTES.get(args.workload, ""),
                       "density": DENSITY, "momentum": MOMENTUM, "policy": args.policy,
                       "asq": bool(args.asq)},
            "cpu_baseline": cb,
            "e2e": {"value": ms_iter, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- GPU arm
class stdout_to_stderr:
    """Redirect file descriptor 1 to 2 (C-level writes included) inside the block."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1808_04357_b200 import rgc as R

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    specs, sizes, kinds = layer_specs(args.workload, args.policy, args.asq)
    N = sum(sizes)
    if args.sync_mode == "auto":
        args.sync_mode = "p2p" if world > 1 else "fixed"
    mode = {"fixed": R.RGC_SYNC_FIXED, "sizes_first": R.RGC_SYNC_SIZES_FIRST,
            "p2p": R.RGC_SYNC_P2P, "pull": R.RGC_SYNC_PULL}[args.sync_mode]
    # NCCL prints its banner on stdout when the image sets NCCL_DEBUG=VERSION: keep stdout
    # for the one JSON line by pointing fd 1 at stderr while the communicators come up
    with stdout_to_stderr():
        nb = args.buckets
        if nb > 1 and args.graph:
            raise SystemExit("--graph with --buckets > 1 is not supported")
        if world > 1:
            dist.init_process_group("nccl", device_id=dev)
            obj = [[R.rgc_get_unique_id() for _ in range(nb)] if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            uids = obj[0]
        else:
            uids = [None] * nb

        def make_engine(uids, mode):
            if nb == 1:
                return R.RGC(specs, rank=rank, nranks=world, device=local, uid=uids[0],
                             sync_mode=mode)
            big = max(range(len(sizes)), key=lambda i: sizes[i])
            groups = [[i for i in range(len(sizes)) if i != big], [big]]
            return R.RGCBuckets(specs, groups, rank=rank, nranks=world, device=local, uids=uids,
                                sync_mode=mode, k1_occ=[None, args.k1_occ_big], priority=[-1, 0])
        try:
            eng = make_engine(uids, mode)
        except R.RgcError as e:
            if mode not in R.P2P_MODES:
                raise
            # no peer mappings between these GPUs: the NCCL allgather instead
            print(f"rank {rank}: RGC_SYNC_P2P unavailable ({e}); using RGC_SYNC_FIXED",
                  file=sys.stderr)
            args.sync_mode, mode = "fixed", R.RGC_SYNC_FIXED
            obj = [[R.rgc_get_unique_id() for _ in range(nb)] if rank == 0 else None]
            if world > 1:
                dist.broadcast_object_list(obj, src=0)
            eng = make_engine(obj[0], mode)

    # synthetic inputs resident in HBM: a pool of distinct i.i.d. N(0, 0.01^2) gradient
    # sets per rank (a fresh minibatch gradient every step, so the residual follows the
    # accumulation dynamics of training instead of a fixed repeating pattern)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    nset = args.pool or max(2, min(64, args.warmup + args.steps,
                                   int(args.pool_gb * 1e9 // (4 * N))))
    G = [[device_gradient(n, args.dist, dev, gen) for n in sizes] for _ in range(nset)]
    V = [torch.zeros(n, device=dev) for n in sizes]
    U = [torch.zeros(n, device=dev) for n in sizes]
    O = [torch.empty(n, device=dev) for n in sizes]
    counter = [0]

    ordered = not args.unordered

    def step(i=None):
        eng.step(G[counter[0] % nset], V, U, O, ordered=ordered)
        counter[0] += 1

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = Clocks(local)
    for i in range(max(3, args.warmup)):
        step()
    barrier()
    graphs = None
    if args.graph:
        # one CUDA graph per gradient set (each set's layer table is resident after one
        # eager call, so no copies are captured); needs a small pool (<= 4 table slots)
        if nset > 4:
            raise SystemExit("--graph needs --pool <= 4")
        for i in range(nset):
            step()
        barrier()
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        graphs = []
        with torch.cuda.stream(gs):
            for i in range(nset):
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr, stream=gs):
                    eng.step(G[i], V, U, O, ordered=ordered)
                graphs.append(gr)
        torch.cuda.current_stream().wait_stream(gs)
        for i in range(nset):
            graphs[i].replay()
        barrier()
    per_graph_launches = 0
    if graphs is not None:
        l0 = eng.launch_count()
        step()
        per_graph_launches = eng.launch_count() - l0
        barrier()
    # the timed loop records events around K1 only (the roofline kernel, timed live); the
    # per-phase breakdown comes from a separate loop with events around every phase
    phase_events = not (args.no_phase_events or args.graph)

    def timed_loop(profile):
        eng.profile(profile)
        eng.profile_read()
        l0 = eng.launch_count()
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        clocks.start()
        e0.record(stream)
        for i in range(args.steps):
            if graphs is not None and not profile:
                graphs[i % nset].replay()
            else:
                step()
        e1.record(stream)
        barrier()
        clocks.stop()
        launches = eng.launch_count() - l0
        if graphs is not None and not profile:
            launches = per_graph_launches * args.steps
        phases = eng.profile_read()[0]
        eng.profile(False)
        return e0.elapsed_time(e1), launches, phases

    # K1's events on every K1_EVERY-th step of the timed loop: K1 timed live on its stream over
    # the timed region, while the other steps keep the programmatic-dependent-launch overlap
    # at K1's edges (events on every step cost ~7 us per step)
    K1_EVERY = 4
    ms, launches, phases = timed_loop(K1_EVERY + 1 if phase_events else 0)
    k1_sampled = (args.steps + K1_EVERY - 1) // K1_EVERY
    k1_live = phases["accumulate"] * args.steps / k1_sampled   # per-step sum scale
    _, _, phases = timed_loop(1)             # phase breakdown from a separate profiled loop
    if phase_events:
        phases["accumulate"] = k1_live
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    ph = torch.tensor([phases[k] for k in R.PHASES], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ph, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ms_step = ms / args.steps
    phase_ms = {k: float(v) / args.steps for k, v in zip(R.PHASES, ph.tolist())}
    info = eng.info()
    counts = [int(i["count"]) for i in info]
    # bytes this rank's message carries (header + 8 per pair, 4 per ASQ index), all ranks
    used = eng.message_bytes(counts)
    ub = torch.tensor([float(used)], device=dev, dtype=torch.float64)
    if world > 1:
        ubs = [torch.zeros_like(ub) for _ in range(world)]
        dist.all_gather(ubs, ub)
        used_all = [float(x.item()) for x in ubs]
    else:
        used_all = [float(used)]
    # selection statistics, outside the timed region: every rank's counts ->
    # effective density D_eff = sum_r c_r / (p n) (the cost model's D for threshold search,
    # P:321); union ratio |U_r idx_r| / n from the last step's dense average (its nonzeros:
    # exact unless a sent value is +-0); the paths (flags) are in layer_diag
    ct = torch.tensor(counts, device=dev, dtype=torch.float64)
    if world > 1:
        cts = [torch.zeros_like(ct) for _ in range(world)]
        dist.all_gather(cts, ct)
        csum = sum(cts)
    else:
        csum = ct
    union = [int(torch.count_nonzero(o).item()) for o in O]
    sel_stats = {
        "D_eff_per_layer": [float(c) / (world * n) for c, n in zip(csum.tolist(), sizes)],
        "D_eff": float(csum.sum().item()) / (world * N),
        "union_ratio_per_layer": [u / n for u, n in zip(union, sizes)],
        "union_ratio": sum(union) / N,
        "union_bound": [DENSITY, min(1.0, world * DENSITY)],
    }

    # context, not in `value`: the layers RGC leaves uncompressed (4n <= 128 KB) as
    # one dense NCCL allreduce bucket per iteration (library call, timed on the device)
    dense_small = None
    if world > 1:
        import synth
        ns = synth.SMALL_ELEMENTS.get(args.workload, 0)
        if ns:
            buf = torch.zeros(ns, device=dev)
            for _ in range(5):
                dist.all_reduce(buf)
            barrier()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record()
            for _ in range(20):
                dist.all_reduce(buf)
            d1.record()
            barrier()
            td = torch.tensor([d0.elapsed_time(d1) / 20], device=dev, dtype=torch.float64)
            dist.all_reduce(td, op=dist.ReduceOp.MAX)
            dense_small = {"elements": ns, "ms": float(td.item()),
                           "note": "uncompressed layers (4n <= 128 KB, P:448) as one dense NCCL "
                                   "allreduce bucket; reported separately, not in value"}

    # e2e: the same step through the public API with pinned HOST buffers (H2D grads, D2H result)
    e2e = None
    if not args.no_e2e:
        # end to end through the public API (RGC.step) with the inputs in pinned HOST memory
        # and the dense averaged gradient read back to the host every step.  Serial: copy in,
        # step, copy out on one stream.  Pipelined (the reported value): double-buffered
        # device inputs/outputs, H2D of step i+2 and D2H of step i on two copy streams while
        # step i+1 computes -- PCIe in both directions at once.
        Gh = [g.cpu().pin_memory() for g in G[0]]
        Oh = [[torch.empty(n, dtype=torch.float32).pin_memory() for n in sizes] for _ in range(2)]
        Gd = [[torch.empty(n, device=dev) for n in sizes] for _ in range(2)]
        Od = [[torch.empty(n, device=dev) for n in sizes] for _ in range(2)]
        main = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

        def e2e_serial(steps):
            for i in range(steps):
                for a, h in zip(Gd[0], Gh):
                    a.copy_(h, non_blocking=True)
                eng.step(Gd[0], V, U, Od[0], ordered=ordered)
                for h, o in zip(Oh[0], Od[0]):
                    h.copy_(o, non_blocking=True)

        def e2e_pipelined(steps, start):
            ev_in, ev_out = [None, None], [None, None]
            s_in.wait_event(start)
            for b in range(min(2, steps)):
                with torch.cuda.stream(s_in):
                    for a, h in zip(Gd[b], Gh):
                        a.copy_(h, non_blocking=True)
                    ev_in[b] = torch.cuda.Event()
                    ev_in[b].record(s_in)
            for i in range(steps):
                b = i % 2
                main.wait_event(ev_in[b])
                if ev_out[b] is not None:          # Od[b]'s previous result is on the host
                    main.wait_event(ev_out[b])
                eng.step(Gd[b], V, U, Od[b], ordered=ordered)
                done = torch.cuda.Event()
                done.record(main)
                s_out.wait_event(done)
                with torch.cuda.stream(s_out):
                    for h, o in zip(Oh[b], Od[b]):
                        h.copy_(o, non_blocking=True)
                    ev_out[b] = torch.cuda.Event()
                    ev_out[b].record(s_out)
                if i + 2 < steps:                  # next input into Gd[b] once step i read it
                    s_in.wait_event(done)
                    with torch.cuda.stream(s_in):
                        for a, h in zip(Gd[b], Gh):
                            a.copy_(h, non_blocking=True)
                        ev_in[b] = torch.cuda.Event()
                        ev_in[b].record(s_in)
            for e in ev_out:
                if e is not None:
                    main.wait_event(e)

        def timed(fn, steps):
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(main)
            fn(steps, f0) if fn is e2e_pipelined else fn(steps)
            f1.record(main)
            barrier()
            t = torch.tensor([f0.elapsed_time(f1) / steps], device=dev, dtype=torch.float64)
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())

        e2e_serial(2)
        t_serial = timed(e2e_serial, args.e2e_steps)
        st = torch.cuda.Event()
        st.record(main)
        e2e_pipelined(4, st)
        t_pipe = timed(e2e_pipelined, args.e2e_steps)
        e2e = {"value": t_pipe, "unit": UNIT, "h2d_bytes_per_step": 4 * N,
               "d2h_bytes_per_step": 4 * N, "serial_ms": t_serial,
               "note": "RGC.step (compress, sync, decompress) with pinned host gradients copied "
                       "in and the dense averaged gradient copied out every step; value: "
                       "double-buffered, copies on two streams overlapping the next step "
                       "(serial_ms: one stream)"}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cb = cpu_baseline(sizes, [s.selector for s in specs], quant=[s.quantize for s in specs])

    if rank == 0:
        peak, peak_src = peaks()
        nvl_peak, nvl_src = nvlink_peak()
        k1_ms = phase_ms["accumulate"]
        k1_bytes = 20 * N            # read g, u, V + write u, V
        step_bytes = k1_bytes + 4 * N
        achieved = k1_bytes / (k1_ms * 1e-3) / 1e9
        compress_ms = sum(phase_ms[k] for k in R.PHASES[:5])
        msg_bytes = int(eng.sizes.msg_bytes)
        # what rank 0 receives: the other ranks' used bytes (P2P / sizes-first move exactly
        # these; the fixed-capacity NCCL allgather moves msg_bytes per rank)
        recv = sum(used_all[1:]) if args.sync_mode in ("p2p", "pull", "sizes_first") \
            else (world - 1) * msg_bytes
        line = {
            "metric": METRIC, "value": ms_step, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, "note": CONFIG_NOTES.get(args.workload, ""),
                       "layers": len(sizes), "elements_per_rank": N, "density": DENSITY,
                       "momentum": MOMENTUM, "policy": args.policy, "asq": bool(args.asq),
                       "selectors": "trimmed top-k (Alg.2) for conv, threshold binary search "
                                    "(Alg.3) for fc" if args.policy == "hybrid" else args.policy,
                       "sync": args.sync_mode, "parallelism": f"dp{world}",
                       "cuda_graph": bool(args.graph),
                       "buckets": (args.buckets if args.buckets == 1 else
                                   {"n": args.buckets, "groups": "[every layer but the largest], "
                                    "[the largest]; one RGC context and stream each, forked and "
                                    "joined every step", "k1_ctas_per_sm_big": args.k1_occ_big}),
                       "k1_events_in_timed_loop": (f"every {K1_EVERY}th step" if phase_events
                                                   else False),
                       "phases_from": "a separate loop with events around every phase (K1's "
                                      "time: the timed loop's own events on every "
                                      f"{K1_EVERY}th step)" if phase_events else
                                      "a separate loop with events around every phase",
                       "inputs": f"synthetic {DIST_TXT.get(args.dist, args.dist)} fp32 gradients: {nset} distinct seeded "
                                 "sets per rank resident in HBM (a fresh gradient each step), "
                                 "residual/momentum state carried across steps",
                       "l2": f"working set {12 * N / 1e9:.2f} GB >> 126 MB L2 (no flush needed)",
                       "decompress": "zero fill of the dense outputs (k6_fill, TMA bulk stores) "
                                     "on a high-priority stream: an early part in K1's ramp-down "
                                     "(>= 32 tiles per K1 CTA), the rest forked after K1, "
                                     "streaming under the selection kernels; then the "
                                     + ("unordered atomic" if args.unordered else "rank-ordered")
                                     + " sparse scatter (rgc_decompress_prefill)"},
            "compress_GBps": 4 * N * world / (compress_ms * 1e-3) / 1e9,
            "compress_GBps_per_gpu": 4 * N / (compress_ms * 1e-3) / 1e9,
            "phase_ms": phase_ms,
            "allgather": {"bytes_received_per_rank": recv, "ms": phase_ms["sync"],
                          "GBps_per_rank": (recv / (phase_ms["sync"] * 1e-3) / 1e9)
                          if world > 1 and phase_ms["sync"] > 0 else None,
                          # nccl-tests convention: algbw = gathered bytes / time,
                          # busbw = algbw (p-1)/p
                          "algbw_GBps": (sum(used_all) / (phase_ms["sync"] * 1e-3) / 1e9)
                          if world > 1 and phase_ms["sync"] > 0 else None,
                          "busbw_GBps": (sum(used_all) / (phase_ms["sync"] * 1e-3) / 1e9
                                         * (world - 1) / world)
                          if world > 1 and phase_ms["sync"] > 0 else None,
                          "nvlink_peak_GBps": nvl_peak, "nvlink_peak_source": nvl_src,
                          "nvlink_frac": (recv / (phase_ms["sync"] * 1e-3) / 1e9 / nvl_peak)
                          if world > 1 and phase_ms["sync"] > 0 else None,
                          "note": "bytes rank 0 receives / sync phase time (variable-length "
                                  "payloads, SURVEY 8(d)); the sync phase also absorbs rank skew"
                                  + ("; RGC_SYNC_PULL moves the bytes inside the decompression"
                                     if args.sync_mode == "pull" else "")},
            "message_pairs": counts, "k_total": int(eng.sizes.k_total),
            "message_bytes_per_rank": used_all,
            "selection": sel_stats,
            "dense_small_layers": dense_small,
            "layer_diag": [{"n": s.n, "sel": s.selector, "flags": i["flags"],
                            "count": int(i["count"]), "survivors": int(i["survivors"]),
                            "trim_level": i["trim_level"], "iters": i["iters"]}
                           for s, i in zip(specs, info)],
            "roofline": {"bound": "hbm", "kernel": "k1_accumulate (accumulate + momentum + stats)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic("k1_accumulate"),
                         "algorithmic_bytes_per_launch": k1_bytes, "peak_source": peak_src,
                         "launch_ms": k1_ms,
                         "note": "K1's launch time, live CUDA events; when K1 has >= 32 tiles per CTA "
                                 "the early zero fill (4 B/element of the step's output) streams "
                                 "beside K1's last ~10% of CTAs, inside this window (DESIGN 12b)"},
            # the whole step against its HBM floor: K1's 20 B/element (12 with m = 0) plus the
            # dense output's 4 B/element (the zero fill); the selection's stash traffic and the
            # pairs are < 1 % of it (SURVEY 8(d) floors, DESIGN 6)
            "step_roofline": {"bound": "hbm", "algorithmic_bytes": step_bytes,
                              "floor_ms": step_bytes / (peak * 1e9) * 1e3,
                              "frac": step_bytes / (peak * 1e9) * 1e3 / ms_step,
                              "peak": peak, "unit": "GB/s"},
            "cpu_baseline": cb,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks.result(),
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
