"""Every rgc_sync mode on ONE GPU (nranks = 1), through the public call a user makes
(RGC.step = prefill + compress + sync + decompress), against the CPU oracle.

At nranks = 1 the exchange moves one block: FIXED passes it through, SIZES_FIRST reads
the length elements on the host and copies exactly the used bytes, P2P runs
the push kernel into the local staging area and PULL publishes an epoch and decompresses
from the block in place -- so the sync and exchange kernels of every mode run on a
1-GPU box (the 2- and 4-GPU runs are tests/test_multigpu.py).  Also: the context status
(include/rgc.h rgc_status) reports a non-finite residual in every mode.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from harness import bits, compare_info, spec
from paper_1808_04357_b200 import rgc as R

pytestmark = pytest.mark.gpu

MODES = {"fixed": R.RGC_SYNC_FIXED, "sizes_first": R.RGC_SYNC_SIZES_FIRST,
         "p2p": R.RGC_SYNC_P2P, "pull": R.RGC_SYNC_PULL}


def _specs():
    return [spec(300_001, sel=0), spec(1_000_000, sel=1), spec(65_537, sel=2, interval=3),
            spec(200_003, sel=1, q=1), spec(4097, sel=0, m=0.0)]


def _oracle_step(specs, g, Vo, Uo, sst, asq):
    msgs, infos = [], []
    for l, s in enumerate(specs):
        idx, val, oi = O.compress_layer(g[l], Uo[l], Vo[l], s.momentum, s.density, s.selector,
                                        s.bs_branch, s.trim_eps or 0.2, s.bs_eps or 1e-3,
                                        s.max_count, interval=s.sample_interval, state=sst[l],
                                        asq=asq[l])
        if s.quantize:
            val = np.full(len(idx), oi["qmean"], np.float32)
        msgs.append((idx, val))
        infos.append(oi)
    return msgs, infos


@pytest.mark.parametrize("mode", list(MODES))
def test_sync_mode_one_gpu_matches_oracle(mode):
    specs = _specs()
    dev = torch.device("cuda", 0)
    eng = R.RGC(specs, nranks=1, device=0, sync_mode=MODES[mode], p2p_inspect=True)
    try:
        V = [torch.zeros(s.n, device=dev) for s in specs]
        U = [torch.zeros(s.n, device=dev) if s.momentum else None for s in specs]
        out = [torch.empty(s.n, device=dev) for s in specs]
        Vo = [np.zeros(s.n, np.float32) for s in specs]
        Uo = [np.zeros(s.n, np.float32) if s.momentum else None for s in specs]
        sst = [O.SampleState() for _ in specs]
        asq = [O.AsqState() if s.quantize else None for s in specs]
        for it in range(6):
            g = [synth.gradient(s.n, "gaussian", seed=7, layer=l, it=it) for l, s in enumerate(specs)]
            for o in out:
                o.fill_(float("nan"))
            eng.step([torch.from_numpy(x).to(dev) for x in g], V, U, out)
            torch.cuda.synchronize()
            msgs, infos = _oracle_step(specs, g, Vo, Uo, sst, asq)
            ginfo = eng.info()
            got = eng.messages()[0]        # the exchanged block (gathered / staging / peer)
            for l, s in enumerate(specs):
                w = f"{mode} it={it} layer {l}"
                compare_info(ginfo[l], infos[l], s, w)
                assert np.array_equal(got[l][0], msgs[l][0]), (w, "indices")
                assert np.array_equal(bits(got[l][1]), bits(msgs[l][1])), (w, "values")
                assert np.array_equal(bits(V[l].cpu().numpy()), bits(Vo[l])), (w, "residual")
                want = O.decompress(s.n, [msgs[l]])
                assert np.array_equal(bits(out[l].cpu().numpy()), bits(want)), (w, "decompress")
            if mode in ("p2p", "sizes_first"):   # exactly the used bytes travelled
                used = eng.used_bytes()
                assert used == 4 * eng.header_words() + sum(
                    (4 if s.quantize else 8) * len(m[0]) for s, m in zip(specs, msgs))
            rc, words = eng.status()
            assert rc == R.RGC_OK and words[0] == 0, (mode, words)
    finally:
        eng.close()


@pytest.mark.parametrize("bad", ["inf", "nan"])
@pytest.mark.parametrize("mode", list(MODES))
def test_nonfinite_residual_reported_in_every_mode(mode, bad):
    # the exchange surfaces device status flags.  One layer's gradient holds a
    # non-finite value: that layer sends an empty set (RGC_F_NONFINITE in its info and in
    # the message's status word), the others are unaffected, and the context status
    # reports RGC_ENONFINITE in every sync mode (SIZES_FIRST also from rgc_sync itself)
    specs = [spec(100_000, sel=0), spec(50_000, sel=1)]
    dev = torch.device("cuda", 0)
    eng = R.RGC(specs, nranks=1, device=0, sync_mode=MODES[mode])
    try:
        V = [torch.zeros(s.n, device=dev) for s in specs]
        U = [torch.zeros(s.n, device=dev) for s in specs]
        out = [torch.empty(s.n, device=dev) for s in specs]
        g = [torch.from_numpy(synth.gradient(s.n, "gaussian", seed=3, layer=l)).to(dev)
             for l, s in enumerate(specs)]
        eng.step(g, V, U, out)
        eng.check()                                   # a clean step reports nothing
        g[1][12345] = float(bad)
        raised = None
        try:
            eng.step(g, V, U, out)                    # SIZES_FIRST raises here
            eng.check()                               # the others on the next wait
        except R.RgcError as e:
            raised = e
        assert raised is not None and raised.code == R.RGC_ENONFINITE, (mode, raised)
        info = eng.info()
        assert info[1]["flags"] & R.F_NONFINITE and info[1]["count"] == 0
        assert not (info[0]["flags"] & R.F_NONFINITE) and info[0]["count"] == R.rgc_k(100_000, 0.001)
        rc, words = eng.status()
        assert rc == R.RGC_ENONFINITE and words[0] & R.F_NONFINITE
        # the report stays until cleared (the residual stays non-finite, so it comes back)
        R.rgc_status(eng.ctx, R.RGC_STATUS_CLEAR, raise_on_error=False)
        rc, words = eng.status()
        assert rc == R.RGC_OK and words[0] == 0
    finally:
        eng.close()


def test_graph_captured_table_slots_are_pinned():
    # a captured graph keeps the device address of its layer-table slot; eager
    # calls with other buffers must never evict it (4 slots; RGC_ESTATE once all are held)
    specs = [spec(70_000, sel=0), spec(30_000, sel=1)]
    dev = torch.device("cuda", 0)
    eng = R.RGC(specs, nranks=1, device=0, prefill=False)
    try:
        mk = lambda: [torch.zeros(s.n, device=dev) for s in specs]
        V, U, out = mk(), mk(), mk()
        G = [[torch.from_numpy(synth.gradient(s.n, "gaussian", seed=9, layer=l, it=i)).to(dev)
              for l, s in enumerate(specs)] for i in range(6)]
        eng.step(G[0], V, U, out)
        torch.cuda.synchronize()
        gs = torch.cuda.Stream()
        gs.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(gr, stream=gs):
                eng.step(G[0], V, U, out)
        torch.cuda.current_stream().wait_stream(gs)
        # eager calls with 5 other gradient sets cycle through the remaining slots
        for i in range(1, 6):
            eng.step(G[i], V, U, out)
        torch.cuda.synchronize()
        # the graph still works on G[0]'s buffers: replay == an eager call on a copy of the state
        V2 = [v.clone() for v in V]
        U2 = [u.clone() for u in U]
        gr.replay()
        torch.cuda.synchronize()
        got_V = [v.clone() for v in V]
        got_out = [o.clone() for o in out]
        for v, v2 in zip(V, V2):
            v.copy_(v2)
        for u, u2 in zip(U, U2):
            u.copy_(u2)
        eng.step(G[0], V, U, out)
        torch.cuda.synchronize()
        for a, b in zip(got_V, V):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32))
        for a, b in zip(got_out, out):
            assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    finally:
        eng.close()
