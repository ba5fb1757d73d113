"""NEXT-3 bucketing (synchronise finished layers while others still compute):
RGCBuckets splits one step into buckets of layers, one context and one CUDA stream each
(bench.py --buckets).  The layers are independent, so every bucket's selection, residual,
momentum and decompressed gradient must be the oracle's: the bucketed step over a mixed
layer list is compared with the oracle bit by bit for several steps (warm candidate stash,
sampled-BS reuse steps), with a bucket K1 at a reduced occupancy as bench.py runs it.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from harness import bits, spec
from paper_1808_04357_b200 import rgc as R

pytestmark = pytest.mark.gpu


def test_bucketed_step_matches_oracle():
    specs = [spec(300_001, sel=0), spec(2_000_000, sel=1), spec(65_537, sel=2, interval=3),
             spec(700_001, sel=0), spec(4097, sel=0, m=0.0), spec(1_000_003, sel=1, q=1)]
    groups = [[1, 3], [0, 2, 4, 5]]
    dev = torch.device("cuda", 0)
    eng = R.RGCBuckets(specs, groups, device=0, k1_occ=[2, None], priority=[0, -1])
    V = [torch.zeros(s.n, device=dev) for s in specs]
    U = [torch.zeros(s.n, device=dev) for s in specs]
    out = [torch.empty(s.n, device=dev) for s in specs]
    Vo = [np.zeros(s.n, np.float32) for s in specs]
    Uo = [np.zeros(s.n, np.float32) for s in specs]
    sst = [O.SampleState() for _ in specs]
    asq = [O.AsqState() if s.quantize else None for s in specs]
    try:
        for it in range(6):
            g = [synth.gradient(s.n, "t3", seed=77, layer=l, it=it) for l, s in enumerate(specs)]
            eng.step([torch.from_numpy(x).to(dev) for x in g], V, U, out)
            torch.cuda.synchronize()
            for l, s in enumerate(specs):
                idx, val, oi = O.compress_layer(g[l], Uo[l], Vo[l], s.momentum, s.density,
                                                s.selector, s.bs_branch, s.trim_eps or 0.2,
                                                s.bs_eps or 1e-3, s.max_count,
                                                interval=s.sample_interval, state=sst[l],
                                                asq=asq[l])
                if s.quantize:
                    val = np.full(len(idx), oi["qmean"], np.float32)
                w = f"it={it} layer {l} n={s.n} sel={s.selector}"
                assert np.array_equal(bits(V[l].cpu().numpy()), bits(Vo[l])), (w, "residual")
                assert np.array_equal(bits(U[l].cpu().numpy()), bits(Uo[l])), (w, "momentum")
                want = O.decompress(s.n, [(idx, val)])
                assert np.array_equal(bits(out[l].cpu().numpy()), bits(want)), (w, "decompress")
        eng.check()
    finally:
        eng.close()
