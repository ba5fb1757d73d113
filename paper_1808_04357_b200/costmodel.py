"""The paper's alpha-beta-gamma communication cost model, NEXT-4.

Host-side analysis only (no device work): Eq. (1) for the sparse (Allgather-based)
synchronisation and Eq. (2) for the dense (Rabenseifner) Allreduce, the bandwidth
coefficient behind the paper's two conclusions, and least-squares fits of
the model's parameters to timings measured on B200 (tools/calibrate.py).

    Eq. (1)  T_sparse = T_select + lg(p) alpha + (p-1) (M D) beta + p gamma_1
    Eq. (2)  T_dense  = 2 lg(p) alpha + 2 (p-1)/p M beta + (p-1)/p gamma_2

alpha: latency per message, beta: transfer time per unit, gamma_1: the
cost to decompress one collected sparse message of a size-M layer, gamma_2: the cost
of the reduction for a size-M message, T_select: communication-set
selection.  M and the transferred size can be counted in elements (the
paper's literal terms) or in bytes (a message carries a 4-byte index and a 4-byte
value per element, or only the index under ASQ plus one 4-byte mean).
"""
from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class CostParams:
    alpha: float = 0.0        # seconds per message
    beta: float = 0.0         # seconds per byte (or per element in element mode)
    gamma1: float = 0.0       # seconds to decompress one collected message of a layer
    gamma2: float = 0.0       # seconds for the reduction of a size-M message
    t_select: float = 0.0     # seconds of communication-set selection


def lg(p: int) -> float:
    """lg(p) of recursive doubling / halving (power-of-two process counts)."""
    if p < 1:
        raise ValueError("p >= 1")
    return math.log2(p)


def sparse_units(M: float, D: float, unit: str = "element", quantized: bool = False) -> float:
    """Size of one node's communication-set ("the size of which is M x D").
    unit "element": M*D (the paper's literal term); "byte": 8 bytes per element
    (index + value), or 4 per element + one 4-byte mean under ASQ."""
    if unit == "element":
        return M * D
    if unit == "byte":
        return 4.0 * M * D + 4.0 if quantized else 8.0 * M * D
    raise ValueError(unit)


def dense_units(M: float, unit: str = "element") -> float:
    """Size of a dense layer: M elements, or 4*M bytes of fp32."""
    if unit == "element":
        return M
    if unit == "byte":
        return 4.0 * M
    raise ValueError(unit)


def t_sparse(c: CostParams, p: int, M: float, D: float, unit: str = "element",
             quantized: bool = False) -> float:
    """Eq. (1): T_select + lg(p) alpha + (p-1) (M D) beta + p gamma_1."""
    return (c.t_select + lg(p) * c.alpha + (p - 1) * sparse_units(M, D, unit, quantized) * c.beta
            + p * c.gamma1)


def t_dense(c: CostParams, p: int, M: float, unit: str = "element") -> float:
    """Eq. (2): 2 lg(p) alpha + 2 (p-1)/p M beta + (p-1)/p gamma_2."""
    return 2 * lg(p) * c.alpha + 2 * (p - 1) / p * dense_units(M, unit) * c.beta + (p - 1) / p * c.gamma2


def bandwidth_coefficient(p: int, D: float) -> float:
    """The sparse bandwidth term relative to one dense copy of the layer: (p-1) D.
    P:376-377: "when p is 128, the communication bandwidth for sparse synchronization will
    be 12.8% of dense synchronization" (the formula gives 12.7%; R19); 1.5625%
    "requires 100% bandwidth of dense Allreduce ... on 64 GPUs" (63 * 1.5625% = 98.4%)."""
    return (p - 1) * D


def crossover_density(c: CostParams, p: int, M: float, unit: str = "byte",
                      quantized: bool = False) -> float:
    """The density D at which Eq. (1) equals Eq. (2) (sparse stops paying off); Eq. (1)
    is linear in D, so this is exact.  Returns inf if sparse never loses below D = 1."""
    base = t_sparse(c, p, M, 0.0, unit, quantized)
    slope = t_sparse(c, p, M, 1.0, unit, quantized) - base
    gap = t_dense(c, p, M, unit) - base
    if slope <= 0:
        return math.inf
    return gap / slope


# ------------------------------------------------------------------ fitting
def _lstsq(rows, ys):
    """Non-negative least squares: every parameter of Eq. (1) / Eq. (2) is a latency, an
    inverse bandwidth or a per-byte cost, none of which can be negative (an unconstrained
    fit of noisy timings returned gamma_2 < 0 in round 1).  scipy's nnls on column-scaled
    rows; a parameter the data pins at the bound comes back as exactly 0."""
    import numpy as np
    from scipy.optimize import nnls
    A = np.asarray(rows, np.float64)
    y = np.asarray(ys, np.float64)
    scale = np.abs(A).max(axis=0)
    scale[scale == 0] = 1.0
    x, _ = nnls(A / scale, y)
    return [float(v) for v in x / scale]


def fit_allgather(samples):
    """samples: [(p, bytes per rank, seconds)] of an Allgather -> (alpha, beta) of
    T = lg(p) alpha + (p-1) bytes beta (the transfer part of Eq. (1))."""
    rows = [(lg(p), (p - 1) * b) for p, b, _ in samples]
    a, bt = _lstsq(rows, [t for _, _, t in samples])
    return a, bt


def fit_allreduce(samples, beta=None):
    """samples: [(p, bytes, seconds)] of a dense Allreduce.  Eq. (2) with a reduction cost
    linear in the size (gamma_2 = g2 * bytes): T = 2 lg(p) alpha + 2 (p-1)/p bytes beta +
    (p-1)/p g2 bytes.  The beta and g2 columns are proportional, so they separate only
    with beta known (e.g. from the Allgather fit): returns (alpha, beta, g2); without beta,
    (alpha, beta_eff, 0) with the reduction folded into beta_eff."""
    ys = [t for _, _, t in samples]
    if beta is None:
        rows = [(2 * lg(p), 2 * (p - 1) / p * b) for p, b, _ in samples]
        a, bt = _lstsq(rows, ys)
        return a, bt, 0.0
    rows = [(2 * lg(p), (p - 1) / p * b) for p, b, _ in samples]
    ys = [t - 2 * (p - 1) / p * b * beta for (p, b, _), t in zip(samples, ys)]
    a, g2 = _lstsq(rows, ys)
    return a, beta, g2


def fit_decompress(samples):
    """samples: [(p, seconds)] of the decompression of p collected messages of one layer
    -> (fixed, gamma_1) of T = fixed + p gamma_1 (the p gamma_1 term of Eq. (1))."""
    rows = [(1.0, float(p)) for p, _ in samples]
    f, g1 = _lstsq(rows, [t for _, t in samples])
    return f, g1
