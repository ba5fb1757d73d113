"""NEXT-4: the alpha-beta-gamma cost model of P:314-380 (host-side, no GPU).

Pinned by hand evaluation of Eq. (1)/(2) in exact rationals, the paper's two numeric
statements, the linearity in D (crossover), and parameter recovery
from synthetic timings.
"""
from fractions import Fraction as F

import pytest

from paper_1808_04357_b200 import costmodel as CM


def test_eq1_eq2_hand_evaluated():
    a, b, g1, g2, ts = F(5, 10**6), F(1, 10**9), F(2, 10**6), F(3, 10**6), F(7, 10**5)
    c = CM.CostParams(float(a), float(b), float(g1), float(g2), float(ts))
    for p, lgp in [(1, 0), (2, 1), (8, 3), (64, 6), (128, 7)]:
        for M in (10**6, 102_760_448):
            for D in (F(1, 1000), F(1, 64)):
                want1 = ts + lgp * a + (p - 1) * (M * D) * b + p * g1
                want2 = 2 * lgp * a + 2 * F(p - 1, p) * M * b + F(p - 1, p) * g2
                assert CM.t_sparse(c, p, M, float(D)) == pytest.approx(float(want1), rel=1e-12)
                assert CM.t_dense(c, p, M) == pytest.approx(float(want2), rel=1e-12)


def test_byte_units_and_asq_halving():
    M, D = 10**8, 0.001
    assert CM.sparse_units(M, D, "byte") == 8 * M * D          # index + value per element
    assert CM.sparse_units(M, D, "byte", quantized=True) == 4 * M * D + 4
    r = CM.sparse_units(M, D, "byte", True) / CM.sparse_units(M, D, "byte")
    assert r == pytest.approx(0.5, abs=1e-5)                    # "reduce 1/2 of the bandwidth"
    assert CM.dense_units(M, "byte") == 4 * M


def test_paper_bandwidth_statements():
    # p = 128, D = 0.1% -> (p-1) D = 12.7% (the paper prints 12.8%, R19)
    assert CM.bandwidth_coefficient(128, 0.001) == pytest.approx(0.127)
    # D = 1.5625% on 64 GPUs needs about the dense bandwidth: 63/64 = 98.4%
    assert CM.bandwidth_coefficient(64, 0.015625) == pytest.approx(63 / 64)
    # "proportional to the number of nodes p"
    assert [CM.bandwidth_coefficient(p, 0.001) for p in (2, 4, 8)] == pytest.approx([0.001, 0.003, 0.007])


def test_crossover_density_is_where_the_models_meet():
    c = CM.CostParams(alpha=3e-6, beta=1 / 400e9, gamma1=5e-6, gamma2=2e-5, t_select=1e-4)
    for p in (2, 8, 64):
        for q in (False, True):
            d = CM.crossover_density(c, p, 25_000_000, "byte", q)
            assert CM.t_sparse(c, p, 25_000_000, d, "byte", q) == pytest.approx(
                CM.t_dense(c, p, 25_000_000, "byte"), rel=1e-9)
    # more ranks -> sparse stops paying off at a lower density (the (p-1) M D beta term)
    ds = [CM.crossover_density(c, p, 25_000_000, "byte") for p in (2, 8, 64)]
    assert ds[0] > ds[1] > ds[2]


def test_fits_recover_parameters():
    alpha, beta, g2 = 7e-6, 1 / 600e9, 1 / 3000e9
    ag = [(p, b, CM.lg(p) * alpha + (p - 1) * b * beta) for p in (2, 4, 8) for b in (4e3, 1e5, 3e6)]
    a, bt = CM.fit_allgather(ag)
    assert a == pytest.approx(alpha, rel=1e-6) and bt == pytest.approx(beta, rel=1e-6)
    ar = [(p, b, 2 * CM.lg(p) * alpha + 2 * (p - 1) / p * b * beta + (p - 1) / p * b * g2)
          for p in (2, 4, 8) for b in (1e5, 1e7, 4e8)]
    a, bt, g = CM.fit_allreduce(ar, beta=beta)          # beta from the Allgather fit
    assert a == pytest.approx(alpha, rel=1e-5) and bt == beta
    assert g == pytest.approx(g2, rel=1e-5)
    a, be, g = CM.fit_allreduce(ar)                      # reduction folded into beta
    assert g == 0.0 and be == pytest.approx(beta + g2 / 2, rel=1e-6)
    f, g1 = CM.fit_decompress([(p, 4e-5 + p * 6e-6) for p in (1, 2, 4, 8, 16)])
    assert f == pytest.approx(4e-5) and g1 == pytest.approx(6e-6)


def test_fits_are_non_negative():
    # every fitted quantity is a latency / inverse bandwidth / per-byte cost: noisy timings
    # whose unconstrained least-squares fit has a negative gamma_2 (round 1's calibration)
    # must come back clamped at 0, and a clean fit is unchanged
    beta = 1 / 500e9
    samples = [(p, b, 2 * CM.lg(p) * 20e-6 + 2 * (p - 1) / p * b * beta * 0.97)
               for p in (2, 4) for b in (1e6, 4e6, 16e6, 64e6)]
    a, bt, g2 = CM.fit_allreduce(samples, beta=beta)
    assert a >= 0 and g2 == 0.0
    clean = [(p, b, 2 * CM.lg(p) * 20e-6 + 2 * (p - 1) / p * b * beta + (p - 1) / p * b * 1e-12)
             for p in (2, 4) for b in (1e6, 4e6, 16e6, 64e6)]
    a, bt, g2 = CM.fit_allreduce(clean, beta=beta)
    assert abs(a - 20e-6) < 1e-9 and abs(g2 - 1e-12) < 1e-15
