"""Parity harness: run the CUDA path (through the C ABI) and the CPU oracle on the
same seeded inputs and compare element by element.

Single GPU, p simulated ranks: each rank compresses with its own context
(nranks = 1); the p message blocks are concatenated rank-major exactly as
rgc_sync's allgather lays them out, and a communicator-less context with
nranks = p decompresses them.  The NCCL exchange itself is covered by
tests/test_multigpu.py.
"""
from __future__ import annotations

import os

import numpy as np
import torch

import oracle as O
import synth
from paper_1808_04357_b200 import rgc as R


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def spec(n, D=0.001, m=0.9, sel=0, branch=0, max_count=0, trim_eps=0.0, bs_eps=0.0,
         interval=0, q=0):
    return R.LayerSpec(n=n, density=D, momentum=m, selector=sel, bs_branch=branch,
                       max_count=max_count, trim_eps=trim_eps, bs_eps=bs_eps,
                       sample_interval=interval, quantize=q)


def compare_info(gi, oi, s, where):
    gflags = gi["flags"] & ~R.F_SURV_CAP
    assert gflags == oi["flags"], (where, "flags", hex(gflags), hex(oi["flags"]))
    assert gi["count"] == oi["count"], (where, "count", gi["count"], oi["count"])
    assert gi["emitted"] == gi["count"], (where, "emitted", gi["emitted"], gi["count"])
    assert gi["maxkey"] == oi["maxkey"], (where, "maxkey")
    if oi["flags"] & O.F_NONFINITE:
        return
    assert gi["mean"] == oi["mean"], (where, "mean", gi["mean"], oi["mean"])
    assert gi["iters"] == oi["iters"], (where, "iters", gi["iters"], oi["iters"])
    for j in range(min(gi["iters"], 16)):
        if gi["lb_mask"] >> j & 1:   # bounded step: the GPU knows c >= this, and c >= 2k
            assert oi["level_count"][j] >= gi["level_count"][j] >= 2 * oi.get("k", 0), (where, "lb", j)
        else:
            assert gi["level_count"][j] == oi["level_count"][j], (where, "level_count", j)
        assert bits([gi["level_thresh"][j]])[0] == bits([oi["level_thresh"][j]])[0], (where, "lt", j)
    if s.selector in (1, 2) and not (oi["flags"] & (O.F_EPS_EXACT | O.F_CAP_EXACT | O.F_DEGENERATE)):
        assert bits([gi["threshold"]])[0] == bits([oi["threshold"]])[0], (where, "threshold")
    if s.selector == 0 and not (oi["flags"] & O.F_DEGENERATE):
        assert gi["trim_level"] == oi["trim_level"], (where, "trim_level")
        assert gi["trim_levels"] == oi["trim_levels"], (where, "trim_levels")
        assert gi["survivors"] == oi["survivors"], (where, "survivors")


class Sim:
    """p ranks of RGC state for a layer list, on the GPU and in the oracle."""

    def __init__(self, specs, p=2, dev=0, prefill=False, tables=False):
        self.specs = specs
        self.p = p
        self.prefill = prefill   # rgc_decompress_prefill: zero fill + sparse scatter
        self.dev = torch.device("cuda", dev)
        # tables: the producers are p-rank contexts (no communicator), so each message carries
        # its range table (k_tab), and the decompression reads them (RGC_ASSUME_TAB) instead of
        # deriving every rank's ranges (k6_prep) -- the multi-GPU path, simulated on one GPU
        self.eng = [R.RGC(specs, nranks=p if tables else 1, device=dev) for _ in range(p)]
        if tables:
            os.environ["RGC_ASSUME_TAB"] = "1"
        try:
            self.dec = R.RGC(specs, nranks=p, device=dev) if p > 1 else self.eng[0]
        finally:
            os.environ.pop("RGC_ASSUME_TAB", None)
        z = lambda n: torch.zeros(n, dtype=torch.float32, device=self.dev)
        self.V = [[z(s.n) for s in specs] for _ in range(p)]
        self.U = [[z(s.n) if s.momentum != 0 else None for s in specs] for _ in range(p)]
        self.Vo = [[np.zeros(s.n, np.float32) for s in specs] for _ in range(p)]
        self.Uo = [[np.zeros(s.n, np.float32) if s.momentum != 0 else None for s in specs]
                   for _ in range(p)]
        self.out = [z(s.n) for s in specs]
        self.sst = [[O.SampleState() for s in specs] for _ in range(p)]   # sampled-BS state
        self.asq = [[O.AsqState() if s.quantize else None for s in specs] for _ in range(p)]

    def step(self, grads, check=True, atomic=False, where=""):
        """grads[r][l]: host float32 arrays.  Runs both sides and compares."""
        p, specs = self.p, self.specs
        for o in self.out:                       # stale contents must not survive
            o.fill_(float("nan"))
        if self.prefill and p == 1:
            self.dec.prefill_outputs(self.out)   # forked after K1 of the compress below
        for r in range(p):
            g_dev = [torch.from_numpy(g).to(self.dev) for g in grads[r]]
            self.eng[r].compress(g_dev, self.V[r], self.U[r])
        torch.cuda.synchronize()
        gathered = torch.cat([e.msg for e in self.eng]) if p > 1 else self.eng[0].msg
        if p > 1:
            self.dec.gathered.copy_(gathered)
            if self.prefill:
                self.dec.prefill_outputs(self.out)   # no compress on this context: fill now
        self.dec.decompress(self.out, ordered=not atomic)
        torch.cuda.synchronize()
        # the context status (rgc_status): nothing but non-finite reports (a test may inject
        # those; the oracle side checks the flags), cleared for the next step
        rc, words = self.dec.status()
        assert rc in (R.RGC_OK, R.RGC_ENONFINITE) and words[0] & ~R.F_NONFINITE == 0, \
            (where, "context status", rc, words)
        if rc != R.RGC_OK:
            R.rgc_status(self.dec.ctx, R.RGC_STATUS_CLEAR, raise_on_error=False)
        if not check:
            return
        # oracle side, rank by rank, layer by layer (Alg. 1 inner loop)
        omsgs = [[None] * len(specs) for _ in range(p)]
        for r in range(p):
            ginfo = self.eng[r].info()
            gmsgs = self.eng[r].messages(self.eng[r].msg)[0]
            for l, s in enumerate(specs):
                idx, val, oi = O.compress_layer(grads[r][l], self.Uo[r][l], self.Vo[r][l],
                                                s.momentum, s.density, s.selector, s.bs_branch,
                                                s.trim_eps or 0.2, s.bs_eps or 1e-3, s.max_count,
                                                interval=s.sample_interval,
                                                state=self.sst[r][l], asq=self.asq[r][l])
                if s.quantize:   # ASQ: indices + the quantized mean
                    val = np.full(len(idx), oi["qmean"], np.float32)
                omsgs[r][l] = (idx, val)
                w = f"{where} rank {r} layer {l} n={s.n} sel={s.selector}"
                compare_info(ginfo[l], oi, s, w)
                gi, gv = gmsgs[l]
                assert np.array_equal(gi, idx), (w, "indices", gi[:8], idx[:8])
                assert np.array_equal(bits(gv), bits(val)), (w, "values")
                Vg = self.V[r][l].cpu().numpy()
                assert np.array_equal(bits(Vg), bits(self.Vo[r][l])), (w, "residual")
                if self.U[r][l] is not None:
                    Ug = self.U[r][l].cpu().numpy()
                    assert np.array_equal(bits(Ug), bits(self.Uo[r][l])), (w, "momentum")
        for l, s in enumerate(specs):
            want = O.decompress(s.n, [omsgs[r][l] for r in range(p)])
            got = self.out[l].cpu().numpy()
            w = f"{where} decompress layer {l}"
            if not atomic:
                assert np.array_equal(bits(got), bits(want)), (w, "ordered decompress")
            else:
                # R14: |a-b| <= 1e-6 * sum_r |v_r[i]| elementwise and rel L2 <= 1e-6
                absum = np.zeros(s.n, np.float64)
                for r in range(p):
                    i, v = omsgs[r][l]
                    np.add.at(absum, i.astype(np.int64), np.abs(v.astype(np.float64)))
                d = np.abs(got.astype(np.float64) - want.astype(np.float64))
                assert (d <= 1e-6 * absum + 0.0).all(), (w, "atomic elementwise")
                nb = np.linalg.norm(want.astype(np.float64))
                if nb > 0:
                    assert np.linalg.norm(d) / nb <= 1e-6, (w, "atomic l2")
        return omsgs

    def close(self):
        for e in self.eng:
            e.close()
        if self.p > 1:
            self.dec.close()


def grads_for(specs, p, dist, seed, it):
    if isinstance(dist, str):
        dist = [dist] * len(specs)
    return [[synth.gradient(s.n, dist[l], seed=seed, rank=r, layer=l, it=it)
             for l, s in enumerate(specs)] for r in range(p)]


def run(specs, p=2, iters=3, dist="gaussian", seed=0, atomic=False, where="", prefill=False,
        tables=False):
    sim = Sim(specs, p, prefill=prefill, tables=tables)
    try:
        for it in range(iters):
            sim.step(grads_for(specs, p, dist, seed, it), atomic=atomic,
                     where=f"{where} it={it} dist={dist}")
    finally:
        sim.close()
