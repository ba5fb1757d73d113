"""CUDA path (librgc.so via the C ABI) vs the CPU oracle, element by element.

Bar (north_star): bit-exact selected index sets, counts, residuals, momenta,
compressed values and the rank-ordered decompressed average; the unordered
atomic decompress within 1e-6 relative (R14).
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from harness import Sim, bits, grads_for, run, spec
from paper_1808_04357_b200 import rgc as R

pytestmark = pytest.mark.gpu

SIZES = [1, 31, 4095, 4096, 4097, 65537, 1_000_000]


@pytest.mark.parametrize("sel", [0, 1])
@pytest.mark.parametrize("n", SIZES)
def test_single_layer_sizes(n, sel):
    run([spec(n, sel=sel)], p=2, iters=3, where=f"n={n}")


@pytest.mark.parametrize("sel", [0, 1])
@pytest.mark.parametrize("dist", list(synth.DISTS))
def test_distributions(dist, sel):
    run([spec(200_003, sel=sel)], p=2, iters=3, dist=dist, where=dist)


def test_c1_parity_centrepiece():
    # BASELINE configs[0]: one 1M-element fp32 gradient, D=0.001, 2 ranks, trimmed + BS, 10 its
    run([spec(1_000_000, sel=0), spec(1_000_000, sel=1)], p=2, iters=10, where="C1")


def test_multi_layer_table_mixed():
    specs = [spec(37, sel=0, m=0.0), spec(4096, sel=1), spec(131_073, sel=0),
             spec(1_000_000, sel=1, branch=1), spec(33_278, sel=1, m=0.0),
             spec(262_144, sel=0, D=0.01), spec(9_000, sel=1, D=0.1)]
    run(specs, p=3, iters=4, dist=["gaussian", "t3", "laplace", "gaussian", "cauchy",
                                   "uniform", "sparse"], where="mixed")


@pytest.mark.parametrize("D", [0.01, 0.1, 0.5, 1.0])
@pytest.mark.parametrize("sel", [0, 1])
def test_densities(D, sel):
    run([spec(50_001, D=D, sel=sel)], p=2, iters=3, where=f"D={D}")


@pytest.mark.parametrize("dist", ["gaussian", "t3", "cauchy", "uniform"])
def test_bs_paper_literal_branch(dist):
    run([spec(300_000, sel=1, branch=1)], p=2, iters=3, dist=dist, where="literal")


def test_bs_capacity_fallback_and_eps():
    # max_count == k: every BS set larger than k falls back to the exact top-k (R18)
    k = O.k_of(120_000, 0.001)
    run([spec(120_000, sel=1, max_count=k), spec(120_000, sel=1, bs_eps=0.25),
         spec(120_000, sel=1, bs_eps=2.0 ** -10)], p=2, iters=3, where="cap")


@pytest.mark.parametrize("m", [0.0, 0.9])
def test_sampled_bs(m):
    # NEXT-1: sampled threshold binary search, search every `interval` calls
    specs = [spec(300_001, sel=2, m=m), spec(120_000, sel=2, m=m, interval=2),
             spec(65_537, sel=2, m=m, interval=3, max_count=4 * 66)]
    run(specs, p=2, iters=12, dist=["gaussian", "t3", "laplace"], where=f"sampled m={m}")


def test_sampled_bs_drift():
    # the distribution changes scale mid-run; reuse steps may leave the band
    specs = [spec(200_000, sel=2, m=0.0), spec(200_000, sel=2, m=0.0, interval=4)]
    sim = Sim(specs, p=1)
    try:
        for it in range(9):
            g = grads_for(specs, 1, "gaussian", 31, it)
            if it >= 3:
                g = [[(x * np.float32(10.0)).astype(np.float32) for x in gr] for gr in g]
            sim.step(g, where=f"drift it={it}")
    finally:
        sim.close()


def test_sampled_reuse_over_capacity_selects_from_survivors():
    # momentum-corrected residuals grow between searches, so a reuse step's count at the
    # cached threshold exceeds the capacity (R18: exact top-k, CAP_EXACT).  The exact top-k
    # then runs over the survivors {|V| > t_cached} (K3A -> K45 / K4 + K3B), not over V;
    # bit-exact with the oracle's exact top-k over V on every call
    specs = [spec(1_000_000, sel=2, interval=5), spec(300_007, sel=2, interval=3),
             spec(4_200_000, sel=2, interval=5)]
    sim = Sim(specs, p=1)
    hits = 0
    try:
        for it in range(12):
            sim.step(grads_for(specs, 1, "gaussian", 83, it), where=f"reuse-cap it={it}")
            for i in sim.eng[0].info():
                want = R.F_SAMPLED_REUSE | R.F_CAP_EXACT
                hits += (i["flags"] & want) == want
    finally:
        sim.close()
    assert hits > 0, "no reuse step exceeded the capacity"


def test_candidate_stash_path_used_and_exact():
    # K1's candidate stash {|V| > tau} (tau predicted from the previous call's t_jlo / t_0)
    # replaces K2's and K3's re-reads of V once the residual is warm; bit-exact either way
    specs = [spec(1_000_000, sel=0), spec(1_000_000, sel=1), spec(262_147, sel=1, m=0.0),
             spec(2_359_296, sel=0)]
    sim = Sim(specs, p=2)
    used = [0] * len(specs)
    try:
        for it in range(10):
            sim.step(grads_for(specs, 2, "gaussian", 41, it), where=f"stash it={it}")
            for l, i in enumerate(sim.eng[0].info()):
                used[l] += i["stashed"]
    finally:
        sim.close()
    assert all(u > 0 for u in used), used


def test_stash_prediction_misses_fall_back_exactly():
    # gradient-scale jumps move t_0 / t_jlo away from the predicted stash key: up (the
    # stash overflows) and down (tau above the needed key); both fall back to the V pass
    specs = [spec(1_000_000, sel=0), spec(1_000_000, sel=1), spec(300_000, sel=2, interval=3),
             spec(500_000, sel=1, m=0.0)]
    scale = {3: 30.0, 4: 30.0, 6: 1e-3, 7: 1e-3, 8: 1e-3, 11: 100.0}
    sim = Sim(specs, p=2)
    used = [0] * len(specs)
    try:
        for it in range(14):
            g = grads_for(specs, 2, "gaussian", 59, it)
            f = np.float32(scale.get(it, 1.0))
            g = [[(x * f).astype(np.float32) for x in gr] for gr in g]
            sim.step(g, where=f"stash-miss it={it}")
            for l, i in enumerate(sim.eng[0].info()):
                used[l] += i["stashed"]
    finally:
        sim.close()
    assert all(0 < u < 14 for u in used), used


def test_stash_window_follows_heavy_tailed_max_jumps():
    # Student-t(3) / Cauchy gradients: max|V| jumps by ~2x from call to call, so the Alg.3
    # level scale moves while the selected threshold value drifts slowly.  K1 derives the
    # bounded histogram's lowest level from the stash key (value space); the stash must keep
    # serving K2/K3 on most calls, and every call stays bit-exact with the oracle (the
    # counts below jlo are bounds, a failed bound re-counts over V)
    specs = [spec(2_000_000, sel=1), spec(700_001, sel=1), spec(1_000_000, sel=1, branch=1),
             spec(400_000, sel=1, m=0.0)]
    dists = ["t3", "cauchy", "t3", "t3"]
    sim = Sim(specs, p=2)
    used = [0] * len(specs)
    iters = 14
    try:
        for it in range(iters):
            sim.step(grads_for(specs, 2, dists, 67, it), where=f"heavy-tail stash it={it}")
            for l, i in enumerate(sim.eng[0].info()):
                used[l] += i["stashed"]
    finally:
        sim.close()
    # the first call has no prediction; afterwards the stash serves the Student-t layers on
    # (nearly) every call.  Cauchy (max jumps by orders of magnitude) and the paper-literal
    # branch (often ends in an exact top-k, which does not read the stash) are parity-only.
    assert used[0] >= iters - 3 and used[3] >= iters - 3, used


def test_trim_eps_variants():
    run([spec(150_000, sel=0, trim_eps=0.1), spec(150_000, sel=0, trim_eps=0.5),
         spec(150_000, sel=0, trim_eps=0.07)], p=2, iters=3, dist="t3", where="trim_eps")


@pytest.mark.parametrize("p", [1, 3, 8])
def test_rank_counts_and_atomic(p):
    specs = [spec(100_000, sel=0), spec(70_001, sel=1)]
    run(specs, p=p, iters=2, where=f"p={p}")
    run(specs, p=p, iters=2, atomic=True, where=f"atomic p={p}")


def test_nonfinite_flagged():
    specs = [spec(10_000, sel=1), spec(10_000, sel=0)]
    sim = Sim(specs, p=1)
    try:
        g = grads_for(specs, 1, "gaussian", 0, 0)
        g[0][0][1234] = np.inf
        g[0][1][77] = np.nan
        sim.step(g, check=False)
        st = R.rgc_check(sim.eng[0].ctx, sim.eng[0].msg, 2)
        assert st & R.F_NONFINITE
        info = sim.eng[0].info()
        assert info[0]["flags"] & R.F_NONFINITE and info[0]["count"] == 0
        assert info[1]["flags"] & R.F_NONFINITE and info[1]["count"] == 0
    finally:
        sim.close()


def test_deterministic_repeat():
    specs = [spec(500_000, sel=0), spec(500_000, sel=1)]
    outs = []
    for _ in range(2):
        sim = Sim(specs, p=2)
        try:
            for it in range(3):
                sim.step(grads_for(specs, 2, "t3", 5, it), check=False)
            outs.append([o.cpu().numpy().copy() for o in sim.out] +
                        [v.cpu().numpy().copy() for v in sim.V[0]])
        finally:
            sim.close()
    for a, b in zip(*outs):
        assert np.array_equal(bits(a), bits(b))


def test_layer_validation_errors():
    with pytest.raises(R.RgcError):
        R.RGC([R.LayerSpec(n=0)])
    with pytest.raises(R.RgcError):
        R.RGC([R.LayerSpec(n=100, density=0.0)])
    with pytest.raises(R.RgcError):
        R.RGC([R.LayerSpec(n=100, bs_eps=1e-4, selector=1)])


# ---------------------------------------------------------------- full sizes
@pytest.mark.slow
def test_vgg16_full_size_hybrid():
    # BASELINE configs[2] shapes, the launch configuration bench.py times (hybrid policy)
    sizes, kinds = synth.model_layers("vgg16")
    specs = [spec(n, sel=synth.selector_for("vgg16", k), m=0.9) for n, k in zip(sizes, kinds)]
    run(specs, p=2, iters=2, where="vgg16")


@pytest.mark.slow
@pytest.mark.parametrize("sel", [0, 1])
def test_m1_1e8_single_layer(sel):
    run([spec(100_000_000, sel=sel)], p=1, iters=2, where="M1")


@pytest.mark.slow
def test_resnet50_full_size_trimmed():
    sizes, kinds = synth.model_layers("resnet50")
    specs = [spec(n, sel=0, m=0.9) for n in sizes]
    run(specs, p=2, iters=2, where="resnet50")


@pytest.mark.slow
def test_alexnet_full_size_bs_heavy_tailed():
    # BASELINE configs[3]: AlexNet, threshold binary search on every layer, Student-t(3)
    sizes, kinds = synth.model_layers("alexnet")
    specs = [spec(n, sel=1, m=0.9) for n in sizes]
    run(specs, p=2, iters=3, dist="t3", where="alexnet-t3")


@pytest.mark.slow
def test_lstm_ptb_full_size_bs():
    # BASELINE configs[4]: the PTB LSTM's 15M embedding/softmax and 4 x 9M hidden tensors
    sizes, kinds = synth.model_layers("lstm_ptb")
    specs = [spec(n, sel=synth.selector_for("lstm_ptb", k), m=0.9) for n, k in zip(sizes, kinds)]
    run(specs, p=1, iters=2, where="lstm-ptb")


# ------------------------------------------- decompression prefill (zero fill + scatter)
PREFILL_SPECS = [(1, 0, 0.001), (4097, 1, 0.001), (100_003, 0, 0.001), (70_001, 1, 0.1),
                 (9_000, 0, 1.0), (262_147, 2, 0.001)]


@pytest.mark.parametrize("p", [1, 2, 3, 8])
def test_prefill_fill_and_sparse_scatter(p):
    # rgc_decompress_prefill: k6_fill (TMA bulk zero stores) + k6_scatter1/k6_scatter,
    # bit-identical to the rank-ordered decompression; outputs start as NaN (harness)
    specs = [spec(n, sel=s, D=D) for n, s, D in PREFILL_SPECS]
    run(specs, p=p, iters=3, prefill=True, where=f"prefill p={p}")
    run(specs, p=p, iters=2, prefill=True, atomic=True, where=f"prefill atomic p={p}")


def test_prefill_dense_tiles_many_ranks():
    # D = 1: every index sent by every rank (all entries of a tile share indices)
    specs = [spec(20_000, sel=0, D=1.0), spec(8192 * 3 + 5, sel=1, D=0.5)]
    run(specs, p=5, iters=2, dist="t3", prefill=True, where="prefill dense")


def test_prefill_other_outputs_fall_back():
    # outputs registered but decompress into other buffers: full decompression, and the
    # registered buffers were zeroed (documented in rgc.h)
    specs = [spec(300_000, sel=0), spec(50_000, sel=1)]
    dev = torch.device("cuda", 0)
    eng = R.RGC(specs, nranks=1, device=0)
    try:
        V = [torch.zeros(s.n, device=dev) for s in specs]
        U = [torch.zeros(s.n, device=dev) for s in specs]
        A = [torch.full((s.n,), 7.0, device=dev) for s in specs]
        B = [torch.full((s.n,), float("nan"), device=dev) for s in specs]
        Vo = [np.zeros(s.n, np.float32) for s in specs]
        Uo = [np.zeros(s.n, np.float32) for s in specs]
        g = grads_for(specs, 1, "gaussian", 3, 0)[0]
        eng.prefill_outputs(A)
        eng.compress([torch.from_numpy(x).to(dev) for x in g], V, U)
        eng.sync()
        eng.decompress(B)
        torch.cuda.synchronize()
        for l, s in enumerate(specs):
            idx, val, _ = O.compress_layer(g[l], Uo[l], Vo[l], s.momentum, s.density, s.selector)
            want = O.decompress(s.n, [(idx, val)])
            assert np.array_equal(bits(B[l].cpu().numpy()), bits(want))
            assert not A[l].cpu().numpy().any()
    finally:
        eng.close()


def test_prefill_step_in_cuda_graph():
    # compress (forks the fill after K1) + sync + decompress (joins it) captured in one
    # CUDA graph; replays match eager steps bit for bit
    specs = [spec(1_000_000, sel=0), spec(300_001, sel=1)]
    dev = torch.device("cuda", 0)
    res = []
    for use_graph in (False, True):
        eng = R.RGC(specs, nranks=1, device=0)
        try:
            V = [torch.zeros(s.n, device=dev) for s in specs]
            U = [torch.zeros(s.n, device=dev) for s in specs]
            out = [torch.full((s.n,), float("nan"), device=dev) for s in specs]
            G = [[torch.from_numpy(x).to(dev) for x in grads_for(specs, 1, "gaussian", 9, it)[0]]
                 for it in range(4)]
            Gs = [torch.empty_like(x) for x in G[0]]
            for a, b in zip(Gs, G[0]):
                a.copy_(b)
            eng.step(Gs, V, U, out)          # warm the layer-table slot before capture
            torch.cuda.synchronize()
            if use_graph:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    with torch.cuda.graph(gr, stream=s):
                        eng.step(Gs, V, U, out)
                torch.cuda.current_stream().wait_stream(s)
                torch.cuda.synchronize()
            for it in range(1, 4):
                for a, b in zip(Gs, G[it]):
                    a.copy_(b)
                for o in out:
                    o.fill_(float("nan"))
                if use_graph:
                    gr.replay()
                else:
                    eng.step(Gs, V, U, out)
            torch.cuda.synchronize()
            res.append([o.cpu().numpy().copy() for o in out] + [v.cpu().numpy().copy() for v in V])
        finally:
            eng.close()
    # both runs: 1 warm step + 3 steps (capturing does not execute the step)
    for a, b in zip(*res):
        assert np.array_equal(bits(a), bits(b))


# ---------------------------------------------------------------- NEXT-2: ASQ
@pytest.mark.parametrize("sel", [0, 1])
@pytest.mark.parametrize("n", [1, 31, 4097, 65537, 1_000_000])
def test_asq_sizes(n, sel):
    # ASQ: signed-view selection (R21), alternating phase, mean message (R22)
    run([spec(n, sel=sel, q=1)], p=2, iters=4, where=f"asq n={n}")


@pytest.mark.parametrize("dist", ["gaussian", "t3", "uniform", "sparse", "equal", "zero", "cauchy"])
def test_asq_distributions_mixed_with_plain_layers(dist):
    # plain and ASQ layers interleaved in one message (plain pairs first, ASQ indices after);
    # "uniform" is all-positive: the negative phase sends empty messages
    specs = [spec(200_003, sel=0, q=1), spec(70_001, sel=1), spec(300_000, sel=1, q=1),
             spec(4096, sel=0), spec(100_000, sel=0, q=1, D=0.01)]
    run(specs, p=3, iters=4, dist=dist, where=f"asq mixed {dist}", prefill=True)
    run(specs, p=2, iters=2, dist=dist, where=f"asq mixed atomic {dist}", atomic=True)


def test_asq_exact_fallbacks_short_messages():
    # few elements of a sign: the exact top-k keeps only the phase's sign (K4 / K45 paths,
    # survivor capacity, BS capacity fallback)
    specs = [spec(5000, sel=0, q=1, D=0.5), spec(300_000, sel=1, q=1, max_count=301),
             spec(3_000_000, sel=0, q=1, D=0.05), spec(2000, sel=1, q=1, D=1.0)]
    run(specs, p=2, iters=4, dist="sparse", where="asq fallbacks")
    run(specs, p=2, iters=2, dist="t3", where="asq fallbacks t3")


def test_asq_halves_payload_bytes():
    # under ASQ the payload is the indices plus one value: used bytes of the block
    # = header + 4 bytes per entry (plain: 8 per pair)
    specs_q = [spec(1_000_000, sel=0, q=1), spec(500_000, sel=1, q=1)]
    specs_p = [spec(1_000_000, sel=0), spec(500_000, sel=1)]
    used = {}
    for name, specs in (("asq", specs_q), ("plain", specs_p)):
        sim = Sim(specs, p=1)
        try:
            for it in range(2):
                sim.step(grads_for(specs, 1, "gaussian", 13, it), where=f"bytes {name}")
            e = sim.eng[0]
            cnt = [i["count"] for i in e.info()]
            H = e.header_words()
            used[name] = (e.used_bytes(e.msg), cnt, H)
        finally:
            sim.close()
    ub, cnt, H = used["asq"]
    assert ub == 4 * H + 4 * sum(cnt)
    ubp, cntp, Hp = used["plain"]
    assert ubp == 4 * Hp + 8 * sum(cntp)


@pytest.mark.parametrize("p", [2, 3, 8])
def test_decompress_from_producer_range_tables(p):
    # the multi-GPU decompression path on one GPU: p-rank producer contexts write their
    # message's per-tile range table (k_tab), the decompression reads the p tables instead of
    # deriving the ranges (k6_prep); rank-ordered output bit-exact vs the oracle (R13, R14),
    # ragged and empty layers, ASQ layers (index-only entries) among plain ones
    specs = [spec(1_000_000, sel=0), spec(262_147, sel=1), spec(8191, sel=0, D=0.01),
             spec(300_007, sel=1, q=1), spec(16_385, sel=1, D=0.002), spec(65_536, sel=0, q=1)]
    run(specs, p=p, iters=3, dist=["gaussian", "t3", "laplace", "gaussian", "sparse", "t3"],
        where=f"tables p={p}", prefill=True, tables=True)
