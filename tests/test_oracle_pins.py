"""Pins of the CPU oracle to things other than itself (task ③).

Every check here is fixed by the paper, the mathematics or a worked example:
exact rational arithmetic, brute-force sorting, closed forms, invariants
stated in PAPER.md / SPEC.md, and hand-worked traces in tests/golden/.
No expected value is produced by the CUDA path.
"""
import itertools
import json
import math
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def f32bits(x):
    return struct.unpack("<I", struct.pack("<f", float(x)))[0]


def bits_arr(a):
    return np.asarray(a, np.float32).view(np.uint32)


def rn32(q: Fraction) -> float:
    """Round an exact rational to the nearest float32 (ties to even), returned as float."""
    if q == 0:
        return 0.0
    neg = q < 0
    a = -q if neg else q
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)
    quantum = Fraction(2) ** (e - 23)
    m = a / quantum
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    v = float(fl * quantum)
    assert v < 3.5e38
    return -v if neg else v


# --------------------------------------------------------------------- O1: k
def test_k_closed_form():
    # north_star "exact count k = ceil(D·n)"; exact rational ceiling as the pin
    Ds = [Fraction(1, 1000), Fraction(1, 500), Fraction(1, 100), Fraction(1, 64),
          Fraction(1, 10), Fraction(1, 4), Fraction(1, 1)]
    rng = np.random.default_rng(0)
    ns = [1, 2, 999, 1000, 1001, 4095, 4096, 4097, 1_000_000, 102_760_448, 2_359_296,
          15_000_000, 2**31 - 1] + [int(x) for x in rng.integers(1, 2**31, 200)]
    for D in Ds:
        for n in ns:
            want = max(1, min(n, math.ceil(D * n)))
            assert O.k_of(n, float(D)) == want, (D, n)
    # SURVEY §8(c) O1 table
    assert O.k_of(1_000_000, 0.001) == 1000
    assert O.k_of(102_760_448, 0.001) == 102_761
    assert O.k_of(2_359_296, 0.001) == 2_360
    assert O.k_of(15_000_000, 0.001) == 15_000


# ------------------------------------------------------------ O2: accumulate
def test_accumulate_exact_fma_and_add():
    rng = np.random.default_rng(1)
    n = 3000
    g = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 3, n)).astype(np.float32)
    u = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 3, n)).astype(np.float32)
    V = (rng.standard_normal(n) * 10.0 ** rng.integers(-6, 3, n)).astype(np.float32)
    g[:5] = [1e-40, -1e-41, 3.0, 0.5, -0.0]      # subnormals / signed zero
    m = np.float32(0.9)
    u2, V2 = u.copy(), V.copy()
    O.accumulate(g, u2, V2, float(m))
    M = Fraction(float(m))
    for i in range(n):
        q = M * Fraction(float(u[i])) + Fraction(float(g[i]))
        if q == 0:
            continue
        ue = np.float32(rn32(q))
        assert f32bits(u2[i]) == f32bits(ue), i
        qv = Fraction(float(V[i])) + Fraction(float(ue))
        if qv == 0:
            continue
        assert f32bits(V2[i]) == f32bits(rn32(qv)), i


def test_accumulate_momentum_zero_is_plain_residual_add():
    # S:402 "m=0 -> reduces to plain residual accumulation V+g"; numpy float32 add is IEEE RN
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["momentum"][0]
    g = np.array(ex["g"], np.float32)
    u = np.array(ex["u"], np.float32)
    V = np.array(ex["V"], np.float32)
    O.accumulate(g, u, V, 0.0)
    assert V.tolist() == ex["V_out"] and u.tolist() == ex["u_out"]
    rng = np.random.default_rng(2)
    g = rng.standard_normal(10000).astype(np.float32)
    V = rng.standard_normal(10000).astype(np.float32)
    want = (V + g).astype(np.float32)
    O.accumulate(g, None, V, 0.0)
    assert np.array_equal(bits_arr(V), bits_arr(want))


def test_scalar_trace_momentum_masking():
    # S:404 scalar trace: m=0.9, g=1 each step; DGC masking zeroes u and V when sent
    g = np.ones(1, np.float32)
    u = np.zeros(1, np.float32)
    V = np.zeros(1, np.float32)
    seq = []
    for step in range(4):
        Vc, uc = V.copy(), u.copy()
        O.accumulate(g, uc, Vc, 0.9)
        seq.append((float(uc[0]), float(Vc[0])))
        if abs(Vc[0]) > 2:                  # hand "select when |V| > 2"
            Vc[:] = 0
            uc[:] = 0
        u, V = uc, Vc
    f = lambda x: float(np.float32(x))
    u1 = 1.0
    u2 = f(f(0.9) * u1 + 1)                 # exact: 0.9f*1 + 1 rounded once
    assert seq[0] == (1.0, 1.0)
    assert seq[1][0] == u2 and seq[1][1] == f(1.0 + u2)
    assert seq[2] == (1.0, 1.0)             # masked at step 2 (|V| = 2.9 > 2)


# ----------------------------------------------------------------- O3: stats
def test_stats_examples():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["stats"]
    for e in ex:
        bad, mk, mean, _ = O.stats(np.array(e["x"], np.float32))
        assert not bad
        assert struct.unpack("<f", struct.pack("<I", mk))[0] == e["max"]
        assert mean == e["mean"], e["cite"]


@pytest.mark.parametrize("dist", ["gaussian", "uniform", "t3", "cauchy", "sparse", "subnormal",
                                  "laplace"])
def test_stats_mean_within_bound_of_exact_rational_mean(dist):
    n = 20000 + 123
    x = synth.gradient(n, dist, seed=3)
    bad, mk, mean, _ = O.stats(x)
    assert not bad
    a = np.abs(x.astype(np.float64))
    assert mk == f32bits(a.max())           # max: brute force
    exact = sum((Fraction(float(v)) for v in a), Fraction(0)) / n
    mx = Fraction(float(a.max()))
    # every mean_fx term truncates < 2^(E_t-30) <= 2^-30 * max; combine in double
    err = abs(Fraction(mean) - exact)
    assert err <= mx / 2**30 + exact / 10**12, (dist, float(err), float(mx))
    assert Fraction(mean) <= exact + exact / 10**12       # truncation never overshoots


def test_stats_order_independent_within_tiles_and_equal_magnitudes():
    rng = np.random.default_rng(4)
    n = 4096 * 3 + 77
    x = (rng.standard_normal(n) * 0.01).astype(np.float32)
    _, mk0, mean0, bins0 = O.stats(x)
    y = x.copy()
    for t0 in range(0, n, 4096):
        seg = y[t0:t0 + 4096]
        rng.shuffle(seg)
        y[t0:t0 + 4096] = seg
    y *= np.where(rng.random(n) < 0.5, -1, 1).astype(np.float32)
    _, mk1, mean1, bins1 = O.stats(y)
    assert mk0 == mk1 and mean0 == mean1 and np.array_equal(bins0, bins1)
    z = np.full(9999, -0.3, np.float32)
    _, mk, mean, _ = O.stats(z)
    assert mean == float(np.float32(0.3)) and mk == f32bits(np.float32(0.3))


def test_mean_fx_hand_worked_bins():
    # R2 pinned by hand-worked bin vectors (tests/golden/mean_fx_bins.json): E_t = floor(log2
    # tile max) for normal and subnormal tiles, floor truncation of each term, the ascending
    # double combine and the final division
    g = json.load(open(os.path.join(GOLD, "mean_fx_bins.json")))
    for c in g["cases"]:
        x = np.zeros(c["n"], np.float32)
        xb = x.view(np.uint32)
        for i, b in c["x_bits"].items():
            xb[int(i)] = int(b, 16)
        bad, mk, mean, bins = O.stats(x)
        assert not bad
        assert mk == int(c["maxkey"], 16), c["name"]
        want = np.zeros(277, np.uint64)
        for e, v in c["bins"].items():
            want[int(e) + 149] = v
        assert np.array_equal(bins, want), (c["name"], {i - 149: int(v) for i, v in enumerate(bins) if v})
        assert mean == float.fromhex(c["mean_hex"]), (c["name"], mean.hex())


@pytest.mark.parametrize("E", [-140, -20, 0, 7, 60])
def test_mean_fx_exact_on_the_quantum_grid(E):
    # closed form: when every |x| of a tile is a multiple of its quantum 2^(E_t - 30), no
    # term truncates and mean_fx is the correctly rounded exact mean RN64(sum|x| / n)
    rng = np.random.default_rng(1000 + E)
    for trial in range(20):
        n = int(rng.integers(2, 4097))
        q = Fraction(2) ** (E - 30)
        # magnitudes m * 2^(E-30) with m < 2^31 (so < 2^(E+1)); one element sets the max
        # in [2^E, 2^(E+1)); the f32 grid limits m to 24 significant bits
        m = rng.integers(0, 2**31, n, dtype=np.int64)
        m[rng.integers(0, n)] = int(rng.integers(2**30, 2**31))
        vals = []
        for mi in m.tolist():
            mi = int(mi)
            sh = max(0, mi.bit_length() - 24)
            if E - 30 + sh < -149:        # below the subnormal grid
                sh = -149 - (E - 30)
            mi = (mi >> sh) << sh
            vals.append(mi)
        mx = max(vals)
        if mx < 2**30:
            continue
        x = np.array([float(Fraction(v) * q) for v in vals], np.float32)
        assert all(Fraction(float(a)) == Fraction(v) * q for a, v in zip(x, vals))
        x *= np.where(rng.random(n) < 0.5, -1, 1).astype(np.float32)
        _, mk, mean, bins = O.stats(x)
        exact = sum((Fraction(v) for v in vals), Fraction(0)) * q / n
        assert mean == float(exact), (E, n, mean, float(exact))
        assert int(bins[E + 149]) == sum(vals)
    # the smallest pair: [1.0, 2^-30] -> (1 + 2^-30) / 2 exactly (one unit of the quantum)
    _, _, mean, _ = O.stats(np.array([1.0, 2.0 ** -30], np.float32))
    assert mean == 0.5 + 2.0 ** -31


def test_stats_nonfinite_flagged():
    x = np.zeros(5000, np.float32)
    x[4097] = np.inf
    assert O.stats(x)[0]
    x[4097] = np.nan
    assert O.stats(x)[0]


# ------------------------------------------------------- count / compaction
def test_count_and_compact_examples():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in ex["count_above"]:
        assert O.count_above(np.array(e["x"], np.float32), e["t"]) == e["count"], e["cite"]
    for e in ex["compact_above"]:
        assert O.nonzero_indices(np.array(e["x"], np.float32), e["t"]).tolist() == e["idx"]
    rng = np.random.default_rng(5)
    x = rng.standard_normal(5000).astype(np.float32)
    for t in [0.0, 0.5, 1.0, 2.5, 10.0]:
        brute = [i for i in range(x.size) if abs(float(x[i])) > np.float32(t)]
        assert O.nonzero_indices(x, t).tolist() == brute
        assert O.count_above(x, t) == len(brute)


# ------------------------------------------------------------ O7: exact top-k
def brute_topk(x, k):
    order = sorted(range(len(x)), key=lambda i: (-abs(float(x[i])), i))
    return sorted(order[:k])


def test_exact_topk_spec_examples():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for e in ex["exact_topk"]:
        x = np.array(e["x"], np.float32)
        idx = O.exact_topk(x, e["k"])
        assert idx.tolist() == e["idx"], e["cite"]
        assert x[idx].tolist() == e["val"]


def test_exact_topk_exhaustive_small_alphabet():
    alphabet = [0.0, 1.0, -1.0, 2.0, -2.0, 3.0, -3.0]
    for n in range(1, 6):
        for tup in itertools.product(alphabet, repeat=n):
            x = np.array(tup, np.float32)
            for k in range(1, n + 1):
                assert O.exact_topk(x, k).tolist() == brute_topk(tup, k)


def test_exact_topk_random_against_full_sort():
    rng = np.random.default_rng(6)
    for trial in range(60):
        n = int(rng.integers(1, 4097))
        x = (rng.standard_normal(n) * rng.choice([1, 1e-3])).astype(np.float32)
        if trial % 3 == 0:
            x = np.round(x * 4).astype(np.float32)            # many ties
        k = int(rng.integers(1, n + 1))
        a = np.abs(x)
        order = np.lexsort((np.arange(n), -a.astype(np.float64)))
        assert O.exact_topk(x, k).tolist() == sorted(order[:k].tolist())


# ----------------------------------------------------- O5: trimmed (Alg. 2)
def test_trimmed_levels_closed_form():
    # ratio 0.8, 0.6, 0.4, 0.2, ~0 (eps = 0.2) -> 5 levels with ratio > 0
    assert O.trim_levels(0.2) == 5
    assert O.trim_levels(0.25) == 3   # 0.75, 0.5, 0.25 (exact dyadics, next is 0)
    assert O.trim_levels(0.5) == 1


def test_trimmed_spec_example_and_exhaustive_oracle_eq():
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["trimmed"][0]
    x = np.array(ex["x"], np.float32)
    _, mk, mean, _ = O.stats(x)
    idx, _ = O.trimmed(x, ex["k"], mean, struct.unpack("<f", struct.pack("<I", mk))[0])
    assert idx.tolist() == ex["idx"]
    # ORACLE-EQ exhaustively on a small alphabet
    alphabet = [0.0, 1.0, -1.0, 2.0, -3.0, 3.0]
    for n in range(1, 5):
        for tup in itertools.product(alphabet, repeat=n):
            x = np.array(tup, np.float32)
            _, mk, mean, _ = O.stats(x)
            mx = struct.unpack("<f", struct.pack("<I", mk))[0]
            for k in range(1, n + 1):
                idx, info = O.trimmed(x, k, mean, mx)
                assert idx.tolist() == brute_topk(tup, k)


@pytest.mark.parametrize("dist", ["gaussian", "uniform", "t3", "cauchy", "sparse", "ties",
                                  "laplace"])
def test_trimmed_equals_full_sort_and_pass_bound(dist):
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 6000))
        x = synth.gradient(n, dist, seed=trial)
        k = int(rng.integers(1, max(2, n // 50) + 1))
        k = min(k, n)
        _, mk, mean, _ = O.stats(x)
        mx = struct.unpack("<f", struct.pack("<I", mk))[0]
        idx, info = O.trimmed(x, k, mean, mx)
        a = np.abs(x)
        order = np.lexsort((np.arange(n), -a.astype(np.float64)))
        assert idx.tolist() == sorted(order[:k].tolist())
        # PASS-BOUND and level semantics: the chosen level is the first with nnz >= k
        assert info["iters"] <= math.ceil(0.8 / 0.2) + 3
        for j in range(info["iters"]):
            t = np.float32(info["level_thresh"][j])
            assert info["level_count"][j] == int((a > t).sum())
            if j > 0:
                assert info["level_thresh"][j] <= info["level_thresh"][j - 1]
        if not info["flags"] & O.F_TRIM_ALL:
            j = info["trim_level"]
            assert info["level_count"][j] >= k
            assert all(info["level_count"][i] < k for i in range(j))
            assert info["survivors"] == info["level_count"][j]


# ------------------------------------------------------- O6: BS (Alg. 3)
FLAGNAMES = {"BS_BREAK": O.F_BS_BREAK, "EPS_KEEP": O.F_EPS_KEEP, "EPS_HIGH": O.F_EPS_HIGH,
             "EPS_BEST": O.F_EPS_BEST, "EPS_EXACT": O.F_EPS_EXACT, "CAP_EXACT": O.F_CAP_EXACT}


def test_bs_hand_worked_paths():
    g = json.load(open(os.path.join(GOLD, "bs_hand_paths.json")))
    for c in g["cases"]:
        x = np.array(c["x"], np.float32)
        bad, mk, mean, _ = O.stats(x)
        assert mean == c["mean"], c["name"]
        assert struct.unpack("<f", struct.pack("<I", mk))[0] == c["max"]
        idx, info = O.bs(x, c["k"], mean, c["max"], 1e-3, c["branch"])
        want = 0
        for f in c["flags"]:
            want |= FLAGNAMES[f]
        assert info["flags"] == want, c["name"]
        assert idx.tolist() == c["idx"], c["name"]
        assert info["count"] == c["count"]
        if "path" in c:
            assert info["iters"] == len(c["path"])
            for j, (_, t, cnt) in enumerate(c["path"]):
                assert info["level_thresh"][j] == t, (c["name"], j)
                assert info["level_count"][j] == cnt, (c["name"], j)
                if "path_bits" in c:   # R3: the exact f32 bits of every threshold
                    assert f32bits(info["level_thresh"][j]) == int(c["path_bits"][j], 16)
            if "threshold" in c:
                assert info["threshold"] == c["threshold"]
        if "counts" in c:
            assert info["level_count"][:len(c["counts"])] == c["counts"], c["name"]


@pytest.mark.parametrize("branch", [0, 1])
@pytest.mark.parametrize("dist", ["gaussian", "uniform", "t3", "cauchy", "laplace", "sparse"])
def test_bs_invariants(dist, branch):
    rng = np.random.default_rng(8)
    for trial in range(25):
        n = int(rng.integers(1000, 40000))
        x = synth.gradient(n, dist, seed=100 + trial)
        k = max(1, n // 1000 * int(rng.integers(1, 4)))
        _, mk, mean, _ = O.stats(x)
        mx = struct.unpack("<f", struct.pack("<I", mk))[0]
        idx, info = O.bs(x, k, mean, mx, 1e-3, branch)
        a = np.abs(x)
        fl = info["flags"]
        assert info["iters"] <= 10                       # eps = 1e-3 -> at most 10 levels
        for j in range(min(info["iters"], 16)):          # every recorded count is a true count
            assert info["level_count"][j] == int((a > np.float32(info["level_thresh"][j])).sum())
        kth = np.sort(a)[::-1][k - 1]
        if fl & (O.F_EPS_EXACT | O.F_CAP_EXACT):
            order = np.lexsort((np.arange(n), -a.astype(np.float64)))
            assert idx.tolist() == sorted(order[:k].tolist())
            continue
        t = np.float32(info["threshold"])
        sel = np.zeros(n, bool)
        sel[idx] = True
        # THRESH-CONSISTENT
        assert (a[sel] > t).all() and not (a[~sel] > t).any()
        assert np.all(np.diff(idx.astype(np.int64)) > 0)
        c = idx.size
        assert c >= k                                    # "at least 0.1% largest"
        assert (a[a > kth] > t).all()                    # BS-CONTAINMENT
        if fl & O.F_BS_BREAK:
            assert k < c < 2 * k                         # band
        assert c <= 2 * k or False is bool(fl & O.F_BS_BREAK)


def test_bs_monotone_hits_band_on_gaussian():
    # R7 evidence (SURVEY §8(c) point 7): the monotone reading reaches the stated band
    hits = 0
    for s in range(8):
        x = synth.gradient(1_000_000, "gaussian", seed=s)
        _, mk, mean, _ = O.stats(x)
        mx = struct.unpack("<f", struct.pack("<I", mk))[0]
        _, info = O.bs(x, 1000, mean, mx, 1e-3, 0)
        hits += bool(info["flags"] & O.F_BS_BREAK)
    assert hits == 8


# ------------------------------------------- O2..O9: one layer of Alg. 1
@pytest.mark.parametrize("selector", [0, 1])
@pytest.mark.parametrize("dist", ["gaussian", "t3", "sparse", "equal", "zero", "ties"])
def test_compress_layer_conservation(selector, dist):
    # ERROR-FEEDBACK CONSERVATION: V_acc == sent + V_new; values bit-identical
    n = 50_000 + 17
    rng = np.random.default_rng(9)
    u = np.zeros(n, np.float32)
    V = np.zeros(n, np.float32)
    for it in range(3):
        g = synth.gradient(n, dist, seed=11, it=it)
        ua, Va = u.copy(), V.copy()
        O.accumulate(g, ua, Va, 0.9)
        idx, val, info = O.compress_layer(g, u, V, 0.9, 0.001, selector)
        k = info["k"]
        assert k == 51
        assert np.all(np.diff(idx.astype(np.int64)) > 0)
        assert np.array_equal(bits_arr(val), bits_arr(Va[idx]))
        mask = np.zeros(n, bool)
        mask[idx] = True
        assert np.array_equal(bits_arr(V[~mask]), bits_arr(Va[~mask]))
        assert np.array_equal(bits_arr(u[~mask]), bits_arr(ua[~mask]))
        assert (bits_arr(V[mask]) == 0).all() and (bits_arr(u[mask]) == 0).all()
        if selector == 0 or info["flags"] & (O.F_DEGENERATE | O.F_CAP_EXACT | O.F_EPS_EXACT):
            assert idx.size == k                         # exact count k (north_star)
            assert idx.tolist() == brute_topk_np(Va, k)
        if dist == "zero" or (dist == "equal" and it == 0):
            assert info["flags"] & O.F_DEGENERATE
            assert idx.tolist() == list(range(k))        # lowest indices win ties (R6)


def brute_topk_np(x, k):
    a = np.abs(x).astype(np.float64)
    order = np.lexsort((np.arange(x.size), -a))
    return sorted(order[:k].tolist())


def test_select_all_identity():
    # masks select everything -> u' == 0 and V' == 0 (D = 1)
    e = json.load(open(os.path.join(GOLD, "spec_examples.json")))["momentum"][1]
    g = np.array(e["g"], np.float32)
    u = np.array(e["u"], np.float32)
    V = np.array(e["V"], np.float32)
    idx, val, info = O.compress_layer(g, u, V, e["m"], e["D"], 0)
    assert idx.tolist() == e["sent_idx"] and val.tolist() == e["sent_val"]
    assert u.tolist() == e["u_after"] and V.tolist() == e["V_after"]


# ------------------------------------------------------- O11: decompress
def test_decompress_examples():
    for e in json.load(open(os.path.join(GOLD, "spec_examples.json")))["scatter_add"]:
        msgs = [(np.array(i, np.uint32), np.array(v, np.float32)) for i, v in e["msgs"]]
        assert O.decompress(e["n"], msgs).tolist() == e["out"], e["cite"]


def test_decompress_dense_equivalence_and_scale():
    # D = 1 equivalence: every rank sends every index -> the rank-ordered dense mean
    rng = np.random.default_rng(10)
    n = 7777
    for p in (1, 2, 3, 4, 8):
        xs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
        msgs = [(np.arange(n, dtype=np.uint32), x) for x in xs]
        acc = np.zeros(n, np.float32)
        for x in xs:
            acc = (acc + x).astype(np.float32)
        want = (acc * np.float32(np.float32(1.0) / np.float32(p))).astype(np.float32)
        got = O.decompress(n, msgs)
        assert np.array_equal(bits_arr(got), bits_arr(want)), p


def test_decompress_sparse_equals_dense_and_union_bound():
    # SPARSE == DENSE and UNION-RATIO in [D, min(1, pD)]
    rng = np.random.default_rng(11)
    n, p, k = 20000, 4, 20
    msgs, dense = [], []
    for r in range(p):
        idx = np.sort(rng.choice(n, k, replace=False)).astype(np.uint32)
        val = rng.standard_normal(k).astype(np.float32)
        msgs.append((idx, val))
        d = np.zeros(n, np.float32)
        d[idx] = val
        dense.append(d)
    acc = np.zeros(n, np.float32)
    for d in dense:
        acc = (acc + d).astype(np.float32)
    want = acc * np.float32(0.25)
    assert np.array_equal(bits_arr(O.decompress(n, msgs)), bits_arr(want))
    union = len(set(np.concatenate([m[0] for m in msgs]).tolist())) / n
    assert k / n <= union <= min(1.0, p * k / n)


# -------------------------------------- sampled threshold BS (NEXT-1)
def test_sampled_interval_one_is_plain_bs():
    # sample_interval = 1 -> identical to threshold_binary_search every step
    n = 40_000
    st = O.SampleState()
    Va, ua = np.zeros(n, np.float32), np.zeros(n, np.float32)
    Vb, ub = np.zeros(n, np.float32), np.zeros(n, np.float32)
    for it in range(6):
        g = synth.gradient(n, "t3", seed=21, it=it)
        ia, va, fa = O.compress_layer(g, ua, Va, 0.9, 0.001, O.SEL_SAMPLED, interval=1, state=st)
        ib, vb, fb = O.compress_layer(g, ub, Vb, 0.9, 0.001, O.SEL_BS)
        assert ia.tolist() == ib.tolist() and np.array_equal(bits_arr(va), bits_arr(vb))
        assert fa["flags"] == fb["flags"] and not fa["flags"] & O.F_SAMPLED_REUSE
    assert st.step == 6


def test_sampled_reuse_schedule_and_threshold_consistency():
    # P:199 "the interval of search is empirically set to 5": full searches at steps 0,5,10
    n = 60_000
    st = O.SampleState()
    V, u = np.zeros(n, np.float32), np.zeros(n, np.float32)
    last_t = None
    for it in range(11):
        g = synth.gradient(n, "gaussian", seed=22, it=it)
        Va, ua = V.copy(), u.copy()
        O.accumulate(g, ua, Va, 0.9)
        idx, val, info = O.compress_layer(g, u, V, 0.9, 0.001, O.SEL_SAMPLED, interval=5, state=st)
        reuse = bool(info["flags"] & O.F_SAMPLED_REUSE)
        assert reuse == (it % 5 != 0), it
        a = np.abs(Va)
        if reuse:
            t = np.float32(last_t)
            assert info["iters"] == 1 and info["level_thresh"][0] == last_t
            assert info["level_count"][0] == int((a > t).sum())         # brute recount
            if info["flags"] & O.F_CAP_EXACT:                            # R18 on a reuse step
                assert info["level_count"][0] > 2 * info["k"]
                assert idx.tolist() == brute_topk_np(Va, info["k"])
            else:
                assert info["threshold"] == last_t
                assert idx.tolist() == np.nonzero(a > t)[0].tolist()   # brute force
        else:
            last_t = info["threshold"]
            assert st.valid == 1 and st.t == np.float32(last_t)
        assert st.step == it + 1


def test_sampled_stationary_input_reuse_equals_fresh_search():
    # stationary input -> reuse-step result sets equal fresh-search result sets
    x = synth.gradient(200_000, "gaussian", seed=23)
    _, mk, mean, _ = O.stats(x)
    mx = struct.unpack("<f", struct.pack("<I", mk))[0]
    k = 200
    idx_full, info = O.bs(x, k, mean, mx, 1e-3, 0)
    st = O.SampleState(step=1, valid=1, t=info["threshold"])
    idx_reuse, info_r = O.sampled_reuse(x, k, st)
    assert idx_reuse.tolist() == idx_full.tolist()
    assert info_r["flags"] == O.F_SAMPLED_REUSE


def test_sampled_drift_and_cache_clearing():
    # scale x10 at step 3 -> a reuse step may leave the band; the next search restores it
    n = 50_000
    k = O.k_of(n, 0.001)
    st = O.SampleState()
    V = np.zeros(n, np.float32)
    counts, flags = [], []
    for it in range(6):
        g = synth.gradient(n, "gaussian", seed=24, it=it) * np.float32(10.0 if it >= 3 else 1.0)
        g = g.astype(np.float32)
        idx, val, info = O.compress_layer(g, None, V, 0.0, 0.001, O.SEL_SAMPLED, interval=5, state=st)
        counts.append(info["count"])
        flags.append(info["flags"])
    assert flags[3] & O.F_SAMPLED_REUSE
    assert not (k < counts[3] < 2 * k) or counts[3] > 2 * k or flags[3] & O.F_CAP_EXACT
    assert not flags[5] & O.F_SAMPLED_REUSE and flags[5] & O.F_BS_BREAK
    assert k < counts[5] < 2 * k
    # an exact fallback clears the cache: all-zero data is degenerate -> next call searches
    st2 = O.SampleState()
    Z = np.zeros(1000, np.float32)
    _, _, i0 = O.compress_layer(np.zeros(1000, np.float32), None, Z, 0.0, 0.01, O.SEL_SAMPLED,
                                interval=5, state=st2)
    assert i0["flags"] & O.F_DEGENERATE and st2.valid == 0
    _, _, i1 = O.compress_layer(synth.gradient(1000, "gaussian", seed=1), None, Z, 0.0, 0.01,
                                O.SEL_SAMPLED, interval=5, state=st2)
    assert not i1["flags"] & O.F_SAMPLED_REUSE


# ------------------------------------------------------------ NEXT-2: ASQ
def _asq_brute(V, k, phase):
    """Plain definition: the k largest signed values (phase 0) / k smallest (phase 1),
    restricted to that sign, lower index first on ties; ascending output."""
    x = np.asarray(V, np.float64) * (1.0 if phase == 0 else -1.0)
    cand = [i for i in range(len(x)) if x[i] > 0]
    cand.sort(key=lambda i: (-x[i], i))
    return np.array(sorted(cand[:k]), np.uint32)


def test_asq_spec_examples():
    # ([0.5,-0.9,0.3], k=1, POSITIVE) -> [0] / 0.5; NEGATIVE -> [1] / -0.9
    for ph, want_i, want_v in [(0, [0], 0.5), (1, [1], -0.9)]:
        V = np.array([0.5, -0.9, 0.3], np.float32)
        st = O.AsqState(); st.phase = ph
        idx, val, info = O.compress_layer(np.zeros(3, np.float32), None, V, 0.0, 1 / 3, 0, asq=st)
        assert list(idx) == want_i and info["qmean"] == np.float32(want_v)
        assert st.phase == 1 - ph                      # PHASE-ALTERNATION
    # quantize_mean [2,4] -> 3.0; [-7] -> -7
    assert O.asq_mean(np.array([2, 4], np.float32)) == 3.0
    assert O.asq_mean(np.array([-7], np.float32)) == -7.0
    assert O.asq_mean(np.zeros(0, np.float32)) == 0.0


def test_asq_view_definition():
    x = np.array([0.0, -0.0, 1.5, -2.5, 1e-45, -1e-45, np.float32(3e38), -3e38], np.float32)
    p = O.asq_view(x, 0)
    n = O.asq_view(x, 1)
    assert list(p) == [0, 0, np.float32(1.5), 0, np.float32(1e-45), 0, np.float32(3e38), 0]
    assert list(n) == [0, 0, 0, np.float32(2.5), 0, np.float32(1e-45), 0, np.float32(3e38)]
    assert not np.signbit(p).any() and not np.signbit(n).any()


@pytest.mark.parametrize("selector", [0, 1])
def test_asq_exhaustive_small_alphabet(selector):
    # every vector over {0, +-1, +-2, +-3} of length <= 4 (and every k): the trimmed
    # selection equals the brute-force signed top-k; BS sets are one-signed, contain
    # the brute set when larger (threshold consistency) and respect the fallback rules
    alpha = [0.0, 1.0, -1.0, 2.0, -2.0, 3.0, -3.0]
    for n in range(1, 5):
        for tup in itertools.product(alpha, repeat=n):
            for k in range(1, n + 1):
                for ph in (0, 1):
                    V = np.array(tup, np.float32)
                    st = O.AsqState(); st.phase = ph
                    idx, val, info = O.compress_layer(np.zeros(n, np.float32), None, V, 0.0,
                                                      k / n, selector, asq=st)
                    want = _asq_brute(tup, k, ph)
                    sgn = 1.0 if ph == 0 else -1.0
                    assert all(sgn * float(v) > 0 for v in val), (tup, k, ph)   # ASQ-SIGN
                    if selector == 0 or info["flags"] & (O.F_DEGENERATE | O.F_EPS_EXACT | O.F_CAP_EXACT):
                        assert np.array_equal(idx, want), (tup, k, ph, idx, want)
                    else:
                        t = info["threshold"]
                        xs = np.asarray(tup) * sgn
                        assert np.array_equal(idx, np.nonzero(xs > t)[0].astype(np.uint32))
                        assert set(want.tolist()) <= set(idx.tolist()) or len(idx) < len(want)


@pytest.mark.parametrize("dist", ["gaussian", "t3", "uniform", "laplace"])
@pytest.mark.parametrize("selector", [0, 1])
def test_asq_random_against_brute_and_mean_exact(dist, selector):
    rng = np.random.default_rng(7)
    for trial in range(6):
        n = int(rng.integers(50, 3000))
        g = synth.gradient(n, dist, seed=trial, layer=selector, it=0)
        D = float(rng.choice([0.01, 0.05, 0.2]))
        k = O.k_of(n, D)
        V = np.zeros(n, np.float32)
        u = np.zeros(n, np.float32)
        st = O.AsqState()
        for it in range(4):
            g = synth.gradient(n, dist, seed=trial, layer=selector, it=it)
            Vacc = V.copy(); uacc = u.copy()
            O.accumulate(g, uacc, Vacc, 0.9)
            ph = st.phase
            idx, val, info = O.compress_layer(g, u, V, 0.9, D, selector, asq=st)
            assert info["phase"] == ph and st.phase == 1 - ph
            sgn = 1.0 if ph == 0 else -1.0
            assert np.all(sgn * val.astype(np.float64) > 0)                      # ASQ-SIGN
            assert np.array_equal(bits_arr(val), bits_arr(Vacc[idx]))           # pre-quantization values
            if selector == 0 or info["flags"] & (O.F_DEGENERATE | O.F_TRIM_ALL | O.F_EPS_EXACT | O.F_CAP_EXACT):
                assert np.array_equal(idx, _asq_brute(Vacc, k, ph))
            else:
                xs = O.asq_view(Vacc, ph)
                assert np.array_equal(idx, np.nonzero(xs > np.float32(info["threshold"]))[0])
            # Alg.1 zeroes the selected residual entries, the rest is untouched
            assert np.all(V[idx] == 0) and np.all(u[idx] == 0)
            rest = np.setdiff1d(np.arange(n), idx)
            assert np.array_equal(bits_arr(V[rest]), bits_arr(Vacc[rest]))
            # R22: the quantized value is the mean of the selected values, rounded once
            if len(val):
                exact = sum(Fraction(float(v)) for v in val) / len(val)
                assert info["qmean"] == rn32(exact), (info["qmean"], float(exact))
            else:
                assert info["qmean"] == 0.0


def test_asq_one_signed_layer_sends_short_or_empty_messages():
    # all-positive residual: the NEGATIVE phase has no candidate (empty message, mean 0);
    # a layer with fewer than k positives sends all of them
    n = 1000
    V = np.abs(synth.gradient(n, "gaussian", seed=3)) + np.float32(1e-3)
    st = O.AsqState()
    idx0, val0, i0 = O.compress_layer(np.zeros(n, np.float32), None, V.copy(), 0.0, 0.01, 0, asq=st)
    assert len(idx0) == 10 and i0["qmean"] > 0
    idx1, val1, i1 = O.compress_layer(np.zeros(n, np.float32), None, V.copy(), 0.0, 0.01, 1, asq=st)
    assert len(idx1) == 0 and i1["qmean"] == 0.0 and i1["count"] == 0
    W = -V.copy()
    W[[5, 17, 400]] = [1.0, 2.0, 3.0]
    st = O.AsqState()
    idx2, val2, _ = O.compress_layer(np.zeros(n, np.float32), None, W, 0.0, 0.01, 0, asq=st)
    assert list(idx2) == [5, 17, 400] and list(val2) == [1.0, 2.0, 3.0]


def test_asq_sampled_bs_rejected():
    # P:292 "sampled threshold binary search selection cannot be used with quantization"
    with pytest.raises(ValueError):
        O.compress_layer(np.zeros(10, np.float32), None, np.zeros(10, np.float32), 0.0, 0.1, 2,
                         state=O.SampleState(), asq=O.AsqState())


def test_asq_mean_bins_exact_for_wide_exponent_ranges():
    # values spanning subnormals to large normals: the bin sum is exact, so the mean
    # is the correctly rounded exact mean (pinned by rationals)
    rng = np.random.default_rng(11)
    for trial in range(200):
        c = int(rng.integers(1, 60))
        mags = np.float32(2.0) ** rng.integers(-149, 100, c).astype(np.float32)
        mags = (mags * rng.uniform(1, 2, c).astype(np.float32)).astype(np.float32)
        mags = mags[np.isfinite(mags) & (mags > 0)]
        if mags.size == 0:
            continue
        sgn = -1 if trial % 2 else 1
        val = (sgn * mags).astype(np.float32)
        exact = sum(Fraction(float(v)) for v in val) / len(val)
        assert O.asq_mean(val) == rn32(exact)
