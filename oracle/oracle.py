"""ctypes front-end of the C oracle (``rgc_oracle.c``).  TEST INFRASTRUCTURE ONLY.

Argument marshalling only: every step of the arithmetic lives in the C file,
which cites the PAPER.md passage each function follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rgc_oracle.c")
_LIB = os.path.join(_HERE, "librgc_oracle.so")
_lock = threading.Lock()
_lib = None

# flag bits (must match rgc_oracle.c; documented in DESIGN.md "Flags")
F_DEGENERATE = 1 << 0
F_TRIM_ALL = 1 << 1
F_BS_BREAK = 1 << 2
F_EPS_HIGH = 1 << 3
F_EPS_BEST = 1 << 4
F_EPS_EXACT = 1 << 5
F_CAP_EXACT = 1 << 6
F_NONFINITE = 1 << 7
F_EPS_KEEP = 1 << 8
F_SAMPLED_REUSE = 1 << 9

SEL_TRIMMED = 0
SEL_BS = 1
SEL_SAMPLED = 2
BS_MONOTONE = 0
BS_PAPER_LITERAL = 1
MAX_LEVELS = 16


class SampleState(C.Structure):
    """Per-layer state of the sampled threshold binary search (step, cached threshold)."""
    _fields_ = [("step", C.c_uint64), ("valid", C.c_int32), ("t", C.c_float)]


class AsqState(C.Structure):
    """Per-layer ASQ phase (0: positive / largest k, 1: negative / smallest k)."""
    _fields_ = [("phase", C.c_uint32)]


class Info(C.Structure):
    _fields_ = [
        ("flags", C.c_uint32),
        ("iters", C.c_uint32),
        ("trim_level", C.c_uint32),
        ("trim_levels", C.c_uint32),
        ("count", C.c_uint64),
        ("threshold", C.c_float),
        ("maxkey", C.c_uint32),
        ("mean", C.c_double),
        ("level_count", C.c_uint64 * MAX_LEVELS),
        ("level_thresh", C.c_float * MAX_LEVELS),
        ("survivors", C.c_uint64),
    ]

    def as_dict(self):
        return {
            "flags": self.flags,
            "iters": self.iters,
            "trim_level": self.trim_level,
            "trim_levels": self.trim_levels,
            "count": self.count,
            "threshold": self.threshold,
            "maxkey": self.maxkey,
            "mean": self.mean,
            "level_count": list(self.level_count),
            "level_thresh": list(self.level_thresh),
            "survivors": self.survivors,
        }


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FMA contraction, no fast-math)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math",
           "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = C.CDLL(build())
            _declare(_lib)
    return _lib


def build_variant(src_text: str, out_so: str) -> str:
    """Compile a modified copy of the oracle source (tests/test_oracle_mutations.py: a
    mutant must fail the pins) with the same flags as build()."""
    src = out_so + ".c"
    with open(src, "w") as f:
        f.write(src_text)
    subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math",
                           "-fPIC", "-shared", "-o", out_so, src, "-lm"])
    return out_so


class use_library:
    """Context manager: route every wrapper of this module through another build of the
    oracle (a mutant from build_variant) and restore the real one afterwards."""

    def __init__(self, so_path: str):
        self.so_path = so_path

    def __enter__(self):
        global _lib
        lib()
        self.saved = _lib
        L = C.CDLL(self.so_path)
        _declare(L)
        _lib = L
        return L

    def __exit__(self, *exc):
        global _lib
        _lib = self.saved
        return False


_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


def _declare(L):
    L.rgco_k.restype = C.c_uint64
    L.rgco_k.argtypes = [C.c_uint64, C.c_double]
    L.rgco_accumulate.restype = None
    L.rgco_accumulate.argtypes = [C.c_uint64, _f32p, C.c_void_p, _f32p, C.c_float]
    L.rgco_stats.restype = C.c_int
    L.rgco_stats.argtypes = [C.c_uint64, _f32p, C.POINTER(C.c_uint32),
                             C.POINTER(C.c_double), _u64p]
    L.rgco_count_above.restype = C.c_uint64
    L.rgco_count_above.argtypes = [C.c_uint64, _f32p, C.c_float]
    L.rgco_nonzero_indices.restype = C.c_uint64
    L.rgco_nonzero_indices.argtypes = [C.c_uint64, _f32p, C.c_float, _u32p]
    L.rgco_exact_topk.restype = None
    L.rgco_exact_topk.argtypes = [C.c_uint64, _f32p, C.c_uint64, _u32p]
    L.rgco_trim_levels.restype = C.c_uint32
    L.rgco_trim_levels.argtypes = [C.c_double]
    L.rgco_trimmed.restype = C.c_uint64
    L.rgco_trimmed.argtypes = [C.c_uint64, _f32p, C.c_uint64, C.c_double, C.c_float,
                               C.c_double, _u32p, C.POINTER(Info)]
    L.rgco_bs.restype = C.c_uint64
    L.rgco_bs.argtypes = [C.c_uint64, _f32p, C.c_uint64, C.c_double, C.c_float,
                          C.c_double, C.c_int, C.c_uint64, _u32p, C.POINTER(Info)]
    L.rgco_compress_layer.restype = C.c_int64
    L.rgco_compress_layer.argtypes = [C.c_uint64, _f32p, C.c_void_p, _f32p, C.c_float,
                                      C.c_double, C.c_int, C.c_int, C.c_double, C.c_double,
                                      C.c_uint64, C.c_uint32, C.c_void_p,
                                      _u32p, _f32p, C.POINTER(Info),
                                      C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_float)]
    L.rgco_asq_view.restype = None
    L.rgco_asq_view.argtypes = [C.c_uint64, _f32p, C.c_int, _f32p]
    L.rgco_asq_mean.restype = C.c_float
    L.rgco_asq_mean.argtypes = [C.c_uint64, _f32p]
    L.rgco_sampled_reuse.restype = C.c_uint64
    L.rgco_sampled_reuse.argtypes = [C.c_uint64, _f32p, C.c_uint64, C.c_uint64,
                                     C.POINTER(SampleState), _u32p, C.POINTER(Info)]
    L.rgco_decompress.restype = None
    L.rgco_decompress.argtypes = [C.c_uint64, C.c_int, _u64p, C.c_void_p, C.c_void_p, _f32p]


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a


def k_of(n: int, D: float) -> int:
    """O1: k = ceil(D*n) clamped to [1, n]."""
    return int(lib().rgco_k(n, D))


def accumulate(g, u, V, m: float) -> None:
    """O2 in place on float32 arrays (u may be None when m == 0)."""
    assert V.dtype == np.float32 and V.flags.c_contiguous
    g = _f32(g)
    up = None
    if u is not None:
        assert u.dtype == np.float32 and u.flags.c_contiguous
        up = u.ctypes.data
    if m != 0.0 and up is None:
        raise ValueError("momentum buffer required when m != 0")
    lib().rgco_accumulate(V.size, g, up, V, m)


def stats(V):
    """O3: returns (nonfinite, maxkey, mean_fx, bins[277])."""
    V = _f32(V)
    mk = C.c_uint32(0)
    mean = C.c_double(0.0)
    bins = np.zeros(277, np.uint64)
    bad = lib().rgco_stats(V.size, V, C.byref(mk), C.byref(mean), bins)
    return bool(bad), int(mk.value), float(mean.value), bins


def count_above(X, t: float) -> int:
    X = _f32(X)
    return int(lib().rgco_count_above(X.size, X, np.float32(t)))


def nonzero_indices(X, t: float):
    X = _f32(X)
    out = np.empty(max(X.size, 1), np.uint32)
    c = lib().rgco_nonzero_indices(X.size, X, np.float32(t), out)
    return out[:c].copy()


def exact_topk(X, k: int):
    """O7: the k ascending indices of the exact top-k by (|x| desc, idx asc)."""
    X = _f32(X)
    out = np.empty(max(k, 1), np.uint32)
    lib().rgco_exact_topk(X.size, X, k, out)
    return out[:k].copy()


def trim_levels(eps: float) -> int:
    return int(lib().rgco_trim_levels(eps))


def trimmed(X, k: int, mean: float, maxf: float, eps: float = 0.2):
    X = _f32(X)
    out = np.empty(max(k, 1), np.uint32)
    info = Info()
    c = lib().rgco_trimmed(X.size, X, k, mean, np.float32(maxf), eps, out, C.byref(info))
    return out[:c].copy(), info.as_dict()


def bs(X, k: int, mean: float, maxf: float, eps: float = 1e-3, branch: int = 0,
       max_count: int | None = None):
    X = _f32(X)
    if max_count is None:
        max_count = 2 * k
    out = np.empty(max(X.size, 1), np.uint32)
    info = Info()
    c = lib().rgco_bs(X.size, X, k, mean, np.float32(maxf), eps, branch, max_count, out,
                      C.byref(info))
    return out[:c].copy(), info.as_dict()


def compress_layer(g, u, V, m: float, D: float, selector: int = SEL_TRIMMED,
                   bs_branch: int = BS_MONOTONE, trim_eps: float = 0.2,
                   bs_eps: float = 1e-3, max_count: int = 0, interval: int = 0,
                   state: "SampleState | None" = None, asq: "AsqState | None" = None):
    """One layer of Alg.1's inner loop (O2..O9), in place on V (and u).

    selector 2 (sampled BS) needs a persistent ``SampleState`` in ``state``.
    ``asq``: a persistent ``AsqState`` turns on ASQ: the message is
    (idx, qmean) with info["qmean"]; ``val`` are the selected pre-quantization values.
    Returns (idx uint32[c], val float32[c], info dict); c == -1 means the
    residual is non-finite (idx/val empty).
    """
    if selector == SEL_SAMPLED and state is None:
        raise ValueError("sampled BS needs a SampleState")
    if selector == SEL_SAMPLED and asq is not None:
        raise ValueError("sampled BS cannot be used with quantization (P:292)")
    assert V.dtype == np.float32 and V.flags.c_contiguous
    n = V.size
    g = _f32(g)
    k = k_of(n, D)
    capm = max_count if max_count else (k if selector == SEL_TRIMMED else 2 * k)
    cap = max(capm, k, 1)
    idx = np.empty(cap, np.uint32)
    val = np.empty(cap, np.float32)
    up = None
    if u is not None:
        assert u.dtype == np.float32 and u.flags.c_contiguous
        up = u.ctypes.data
    if m != 0.0 and up is None:
        raise ValueError("momentum buffer required when m != 0")
    info = Info()
    ph = C.c_uint32(asq.phase if asq is not None else 0)
    qm = C.c_float(0.0)
    c = lib().rgco_compress_layer(n, g, up, V, m, D, selector, bs_branch, trim_eps,
                                  bs_eps, max_count, interval,
                                  C.cast(C.pointer(state), C.c_void_p) if state is not None else None,
                                  idx, val, C.byref(info), 1 if asq is not None else 0,
                                  C.byref(ph), C.byref(qm))
    d = info.as_dict()
    d["k"] = k
    if asq is not None:
        d["phase"] = asq.phase          # the phase this call used
        d["qmean"] = float(np.float32(qm.value))
        asq.phase = ph.value
    if c < 0:
        return np.empty(0, np.uint32), np.empty(0, np.float32), d
    return idx[:c].copy(), val[:c].copy(), d


def asq_view(X, phase: int):
    """R21: the signed view of ASQ's phase (0: max(x, 0); 1: max(-x, 0))."""
    X = _f32(X)
    out = np.empty(max(X.size, 1), np.float32)
    lib().rgco_asq_view(X.size, X, phase, out)
    return out[:X.size].copy()


def asq_mean(val) -> float:
    """R22: the quantized value of a one-signed communication-set (0 if empty)."""
    v = _f32(val)
    if v.size == 0:
        v = np.zeros(1, np.float32)
        return float(lib().rgco_asq_mean(0, v))
    return float(np.float32(lib().rgco_asq_mean(v.size, v)))


def sampled_reuse(X, k: int, state: SampleState, max_count: int | None = None):
    """The reuse step of sampled BS on its own: {|x| > state.t} (or exact top-k over capacity)."""
    X = _f32(X)
    if max_count is None:
        max_count = 2 * k
    out = np.empty(max(X.size, 1), np.uint32)
    info = Info()
    c = lib().rgco_sampled_reuse(X.size, X, k, max_count, C.byref(state), out, C.byref(info))
    return out[:c].copy(), info.as_dict()


def decompress(n: int, msgs):
    """O11: msgs = [(idx uint32[], val float32[]) for rank 0..p-1] -> out float32[n]."""
    p = len(msgs)
    counts = np.array([len(i) for i, _ in msgs], np.uint64)
    keep = []
    ip = (C.c_void_p * p)()
    vp = (C.c_void_p * p)()
    for r, (i, v) in enumerate(msgs):
        i = np.ascontiguousarray(i, np.uint32)
        v = np.ascontiguousarray(v, np.float32)
        if i.size == 0:
            i = np.zeros(1, np.uint32)
            v = np.zeros(1, np.float32)
        keep.append((i, v))
        ip[r] = i.ctypes.data
        vp[r] = v.ctypes.data
    out = np.empty(max(n, 1), np.float32)
    lib().rgco_decompress(n, p, counts, C.cast(ip, C.c_void_p), C.cast(vp, C.c_void_p), out)
    return out[:n]
