"""The call bench.py times, at BASELINE.json's full size, against the oracle.

bench.py times RGC.step (decompression prefill, compress, RGC_SYNC_FIXED, decompress) over
the workload's compressed layers with the hybrid policy (trimmed top-k for conv layers,
threshold binary search for fc / LSTM layers, R16), m = 0.9, D = 0.001, a fresh gradient
every step and the residual / momentum state carried across steps.  This test replays that
exact call for WARM_STEPS steps (gradients drawn on the host by synth and uploaded, so the
oracle sees the same arrays) and runs the oracle beside it on every step: every step's
flags, search path, counts, indices and values must match; the residual, momentum and the
dense averaged gradient are compared bitwise on the last two steps.  It also asserts that
the warm-state machinery the bench relies on actually ran -- candidate-stash-served
selections and Alg.3 steps decided by the bounded histogram's lower bound (lb_mask).
"""
import os
import sys

import numpy as np
import pytest
import torch

import oracle as O
import synth
from harness import bits, compare_info
from paper_1808_04357_b200 import rgc as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (layer_specs: the bench's exact layer list)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

WARM_STEPS = 10


@pytest.mark.parametrize("workload,asq", [("vgg16", False), ("m1", False), ("vgg16", True)])
def test_bench_call_warm_full_size(workload, asq):
    # asq: bench.py --asq (P:274-294 on every layer but the output layer)
    specs, sizes, kinds = bench.layer_specs(workload, "hybrid", asq)
    dev = torch.device("cuda", 0)
    eng = R.RGC(specs, nranks=1, device=0, sync_mode=R.RGC_SYNC_FIXED)   # bench at N = 1
    assert eng.prefill
    L = len(specs)
    V = [torch.zeros(n, device=dev) for n in sizes]
    U = [torch.zeros(n, device=dev) for n in sizes]
    out = [torch.empty(n, device=dev) for n in sizes]
    Vo = [np.zeros(n, np.float32) for n in sizes]
    Uo = [np.zeros(n, np.float32) for n in sizes]
    Ao = [O.AsqState() if s.quantize else None for s in specs]
    stashed = lb_steps = 0
    try:
        for it in range(WARM_STEPS):
            g = [synth.gradient(n, "gaussian", seed=2024, layer=l, it=it)
                 for l, n in enumerate(sizes)]
            eng.step([torch.from_numpy(x).to(dev) for x in g], V, U, out)
            ginfo = eng.info()
            got = eng.messages()[0]
            last = it >= WARM_STEPS - 2
            for l, s in enumerate(specs):
                idx, val, oi = O.compress_layer(g[l], Uo[l], Vo[l], s.momentum, s.density,
                                                s.selector, s.bs_branch, 0.2, 1e-3, 0, asq=Ao[l])
                if s.quantize:   # ASQ: indices + the quantized mean
                    val = np.full(len(idx), oi["qmean"], np.float32)
                w = f"{workload} asq={asq} it={it} layer {l} n={s.n} sel={s.selector}"
                compare_info(ginfo[l], oi, s, w)
                assert np.array_equal(got[l][0], idx), (w, "indices")
                assert np.array_equal(bits(got[l][1]), bits(val)), (w, "values")
                stashed += ginfo[l]["stashed"]
                lb_steps += ginfo[l]["lb_mask"] != 0
                if last:
                    assert np.array_equal(bits(V[l].cpu().numpy()), bits(Vo[l])), (w, "residual")
                    assert np.array_equal(bits(U[l].cpu().numpy()), bits(Uo[l])), (w, "momentum")
                    want = O.decompress(s.n, [(idx, val)])
                    assert np.array_equal(bits(out[l].cpu().numpy()), bits(want)), (w, "decompress")
            del g
        eng.check()
    finally:
        eng.close()
    assert stashed > 0, "no selection was served by the K1 candidate stash"
    if any(s.selector == R.RGC_SEL_THRESHOLD_BS for s in specs):
        assert lb_steps > 0, "no Alg.3 step was decided by the bounded histogram's bound"
