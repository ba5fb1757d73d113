"""Thin Python binding of librgc.so (include/rgc.h): argument marshalling only.

Every step of the RGC path runs in the CUDA kernels behind the C ABI; this
module converts torch tensors to device pointers and back.  There is no CPU
fallback: if librgc.so is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RGC_LIB_PATH") or os.path.join(_HERE, "librgc.so")

RGC_OK, RGC_EINVAL, RGC_ECUDA, RGC_ENCCL, RGC_ENONFINITE, RGC_ESTATE = range(6)
RGC_SEL_TRIMMED, RGC_SEL_THRESHOLD_BS, RGC_SEL_SAMPLED_BS = 0, 1, 2
RGC_BS_MONOTONE, RGC_BS_PAPER_LITERAL = 0, 1
RGC_SYNC_FIXED, RGC_SYNC_SIZES_FIRST, RGC_SYNC_P2P, RGC_SYNC_PULL = 0, 1, 2, 3
P2P_MODES = (RGC_SYNC_P2P, RGC_SYNC_PULL)   # both use the rgc_p2p_init block
RGC_MAX_LAYERS = 128
RGC_STATUS_WAIT, RGC_STATUS_CLEAR = 1, 2
STAT_TIMEOUT = 1 << 30          # rgc_status word 0: a cross-GPU wait timed out
RGC_MSG_DENSE = 0xFFFFFFFF     # header value word of a plain (non-ASQ) layer
RGC_NPHASE = 7
PHASES = ("accumulate", "count_search", "compact", "select", "emit", "sync", "decompress")

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
F_SURV_CAP = 1 << 16


class RgcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"rgc error {code}: {msg}")
        self.code = code


class rgc_layer_t(C.Structure):
    _fields_ = [("n", C.c_uint64), ("density", C.c_double), ("momentum", C.c_float),
                ("selector", C.c_int32), ("bs_branch", C.c_int32), ("trim_eps", C.c_double),
                ("bs_eps", C.c_double), ("max_count", C.c_uint32), ("sample_interval", C.c_uint32),
                ("quantize", C.c_int32)]


class rgc_info_t(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("iters", C.c_uint32), ("trim_level", C.c_uint32),
                ("trim_levels", C.c_uint32), ("count", C.c_uint64), ("threshold", C.c_float),
                ("maxkey", C.c_uint32), ("mean", C.c_double),
                ("level_count", C.c_uint64 * 16), ("level_thresh", C.c_float * 16),
                ("survivors", C.c_uint64), ("kth_key", C.c_uint32), ("tie_quota", C.c_uint32),
                ("emitted", C.c_uint64), ("lb_mask", C.c_uint32), ("stashed", C.c_uint32)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["level_count"] = list(self.level_count)
        d["level_thresh"] = list(self.level_thresh)
        return d


class rgc_sizes_t(C.Structure):
    _fields_ = [("workspace_bytes", C.c_uint64), ("msg_bytes", C.c_uint64),
                ("gathered_bytes", C.c_uint64), ("header_bytes", C.c_uint64),
                ("k_total", C.c_uint64), ("cap_total", C.c_uint64)]


_lib = None


def lib():
    """Load librgc.so (no fallback: raises if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_1808_04357_b200.build` (needs nvcc, sm_100a)")
        L = C.CDLL(LIB_PATH)
        vp, i32, u64 = C.c_void_p, C.c_int, C.c_uint64
        sig = {
            "rgc_version": (C.c_char_p, []),
            "rgc_status_string": (C.c_char_p, [i32]),
            "rgc_k": (i32, [u64, C.c_double, C.POINTER(C.c_uint64)]),
            "rgc_get_unique_id": (i32, [C.c_char_p]),
            "rgc_init": (i32, [C.POINTER(vp), i32, i32, i32, C.c_char_p, vp]),
            "rgc_set_stream": (i32, [vp, vp]),
            "rgc_finalize": (i32, [vp]),
            "rgc_last_error": (C.c_char_p, [vp]),
            "rgc_sizes": (i32, [vp, vp, i32, C.POINTER(rgc_sizes_t)]),
            "rgc_workspace_init": (i32, [vp, vp, i32, vp]),
            "rgc_compress": (i32, [vp, vp, i32, vp, vp, vp, vp, vp]),
            "rgc_sync": (i32, [vp, vp, i32, vp, vp, i32, vp]),
            "rgc_decompress": (i32, [vp, vp, i32, vp, vp, i32, vp]),
            "rgc_decompress_prefill": (i32, [vp, vp, i32, vp]),
            "rgc_debug_layer": (i32, [vp, vp, i32, vp, i32]),
            "rgc_get_info": (i32, [vp, i32, vp, C.POINTER(rgc_info_t)]),
            "rgc_check": (i32, [vp, vp, i32, C.POINTER(C.c_uint32)]),
            "rgc_status": (i32, [vp, i32, vp]),
            "rgc_debug_timeline": (i32, [vp, vp, i32]),
            "rgc_profile": (i32, [vp, i32]),
            "rgc_profile_read": (i32, [vp, C.POINTER(C.c_float), i32, C.POINTER(C.c_int)]),
            "rgc_launch_count": (C.c_uint64, [vp]),
            "rgc_sync_plan": (i32, [vp, i32, i32, C.c_uint32, u64, vp, vp, C.POINTER(C.c_uint32)]),
            "rgc_p2p_init": (i32, [vp, vp, i32, C.POINTER(vp)]),
            "rgc_p2p_gather": (i32, [vp, vp, i32, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return [n for n in dir(lib()) if n.startswith("rgc_")]


def _check(rc, ctx=None):
    if rc != RGC_OK:
        msg = lib().rgc_last_error(ctx).decode() if ctx else lib().rgc_status_string(rc).decode()
        raise RgcError(rc, msg)


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _ptrs(ts):
    arr = (C.c_void_p * len(ts))()
    for i, t in enumerate(ts):
        arr[i] = None if t is None else t.data_ptr()
    return arr


# ----------------------------------------------------------- C-ABI names
def rgc_version() -> str:
    return lib().rgc_version().decode()


def rgc_k(n: int, density: float) -> int:
    k = C.c_uint64(0)
    _check(lib().rgc_k(n, density, C.byref(k)))
    return int(k.value)


def rgc_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().rgc_get_unique_id(buf))
    return buf.raw


def rgc_init(rank: int, nranks: int, device: int, uid: bytes | None, stream: int | None):
    ctx = C.c_void_p()
    rc = lib().rgc_init(C.byref(ctx), rank, nranks, device, uid, C.c_void_p(stream or 0))
    _check(rc)
    return ctx


def rgc_set_stream(ctx, stream: int):
    _check(lib().rgc_set_stream(ctx, C.c_void_p(stream)), ctx)


def rgc_finalize(ctx):
    _check(lib().rgc_finalize(ctx))


def make_layers(specs):
    """specs: list of dicts / LayerSpec with n, density, momentum, selector, ..."""
    arr = (rgc_layer_t * len(specs))()
    for i, s in enumerate(specs):
        s = s if isinstance(s, dict) else s.__dict__
        arr[i].n = int(s["n"])
        arr[i].density = float(s.get("density", 0.001))
        arr[i].momentum = float(s.get("momentum", 0.0))
        arr[i].selector = int(s.get("selector", RGC_SEL_TRIMMED))
        arr[i].bs_branch = int(s.get("bs_branch", RGC_BS_MONOTONE))
        arr[i].trim_eps = float(s.get("trim_eps", 0.0))
        arr[i].bs_eps = float(s.get("bs_eps", 0.0))
        arr[i].max_count = int(s.get("max_count", 0))
        arr[i].sample_interval = int(s.get("sample_interval", 0))
        arr[i].quantize = int(s.get("quantize", 0))
    return arr


def rgc_sizes(ctx, layers) -> rgc_sizes_t:
    out = rgc_sizes_t()
    _check(lib().rgc_sizes(ctx, layers, len(layers), C.byref(out)), ctx)
    return out


def rgc_workspace_init(ctx, layers, ws):
    _check(lib().rgc_workspace_init(ctx, layers, len(layers), _ptr(ws)), ctx)


def rgc_compress(ctx, layers, grads, residuals, momenta, msg, ws):
    mom = _ptrs(momenta) if momenta is not None else None
    _check(lib().rgc_compress(ctx, layers, len(layers), _ptrs(grads), _ptrs(residuals), mom,
                              _ptr(msg), _ptr(ws)), ctx)


def rgc_sync(ctx, layers, msg, gathered, mode=RGC_SYNC_FIXED, counts_host=None):
    buf = None
    if counts_host is not None:
        buf = (C.c_uint32 * counts_host.size).from_address(counts_host.ctypes.data)
    rc = lib().rgc_sync(ctx, layers, len(layers), _ptr(msg), _ptr(gathered), mode,
                        C.cast(buf, C.c_void_p) if buf is not None else None)
    _check(rc, ctx)


def rgc_sync_plan(headers, nranks: int, L: int, header_words: int, msg_bytes: int):
    """headers: numpy uint32[nranks*header_words] -> (bytes uint64[nranks], counts uint32[nranks*L], status)"""
    import numpy as np
    h = np.ascontiguousarray(headers, dtype=np.uint32)
    b = np.zeros(nranks, np.uint64)
    cnt = np.zeros(nranks * L, np.uint32)
    st = C.c_uint32(0)
    _check(lib().rgc_sync_plan(h.ctypes.data, nranks, L, header_words, msg_bytes, b.ctypes.data,
                               cnt.ctypes.data, C.byref(st)))
    return b, cnt, int(st.value)


class DevicePtr:
    """A library-owned device block (rgc_p2p_init): exposes data_ptr() like a tensor."""

    def __init__(self, addr: int, nbytes: int):
        self.addr, self.nbytes = int(addr), int(nbytes)

    def data_ptr(self):
        return self.addr


def rgc_p2p_init(ctx, layers, nbytes: int) -> DevicePtr:
    out = C.c_void_p()
    _check(lib().rgc_p2p_init(ctx, layers, len(layers), C.byref(out)), ctx)
    return DevicePtr(out.value, nbytes)


def rgc_p2p_gather(ctx, layers, gathered):
    _check(lib().rgc_p2p_gather(ctx, layers, len(layers), _ptr(gathered)), ctx)


def rgc_decompress(ctx, layers, gathered, outs, ws, ordered=True):
    _check(lib().rgc_decompress(ctx, layers, len(layers), _ptr(gathered), _ptrs(outs),
                                1 if ordered else 0, _ptr(ws)), ctx)


def rgc_decompress_prefill(ctx, layers, outs):
    _check(lib().rgc_decompress_prefill(ctx, layers, len(layers), _ptrs(outs)), ctx)


def rgc_get_info(ctx, L, ws):
    arr = (rgc_info_t * L)()
    _check(lib().rgc_get_info(ctx, L, _ptr(ws), arr), ctx)
    return [a.as_dict() for a in arr]


DEBUG_FIELDS = ("mode", "count", "thr_key", "stash_key", "stash_shift", "stash_on", "stash_ok",
                "k2_from_stash", "k3_from_stash", "need_full", "bs_hint", "bs_margin", "asq_phase",
                "survivors", "emitted_a", "emitted_b", "stash_records",
                "need_count", "vpass_runs", "full_runs")


def rgc_debug_layer(ctx, ws, l: int) -> dict:
    out = (C.c_uint32 * 20)()
    _check(lib().rgc_debug_layer(ctx, _ptr(ws), l, out, 20), ctx)
    return dict(zip(DEBUG_FIELDS, [int(x) for x in out]))


def rgc_check(ctx, msg, L) -> int:
    st = C.c_uint32(0)
    rc = lib().rgc_check(ctx, _ptr(msg), L, C.byref(st))
    if rc not in (RGC_OK, RGC_ENONFINITE):
        _check(rc, ctx)
    return int(st.value)


def rgc_status(ctx, flags=0, raise_on_error=True):
    """Context status (include/rgc.h rgc_status): (rc, [status bits, timeout mask lo, hi,
    NCCL error]).  flags: RGC_STATUS_WAIT / RGC_STATUS_CLEAR; 0 polls without a sync."""
    import numpy as np
    out = np.zeros(4, np.uint32)
    rc = lib().rgc_status(ctx, int(flags), out.ctypes.data)
    if raise_on_error:
        _check(rc, ctx)
    return rc, [int(x) for x in out]


TL_NAMES = ("K1", "K2_stash", "K2_vpass0", "K2_vpass1", "K3A", "K3B", "K45", "K4", "K5",
            "fill", "scatter", "k6_prep", "k_tab", "K6", "K1_stream", "K1_finalize",
            "K2_finalize", "K2_global") + tuple(f"p{i}" for i in range(14))


def rgc_debug_timeline(ctx):
    """{kernel: (start_us, end_us)} of the last step relative to K1's start (contexts created
    with RGC_TIMELINE=1); kernels that did not run are omitted."""
    import numpy as np
    out = np.zeros(64, np.uint64)
    _check(lib().rgc_debug_timeline(ctx, out.ctypes.data, 64), ctx)
    t0 = int(out[0])
    if t0 == 0xFFFFFFFFFFFFFFFF:   # no K1 in the step (a decompression alone): its first kernel
        starts = [int(out[i]) for i in range(len(TL_NAMES)) if int(out[i]) != 0xFFFFFFFFFFFFFFFF]
        t0 = min(starts) if starts else 0
    res = {}
    for i, name in enumerate(TL_NAMES):
        a, b = int(out[i]), int(out[32 + i])
        if a != 0xFFFFFFFFFFFFFFFF and b:
            res[name] = ((a - t0) / 1e3, (b - t0) / 1e3)
    return res


def rgc_profile(ctx, enable):
    """enable: False/0 off, True/1 every phase, 2 the accumulate phase (K1) only."""
    _check(lib().rgc_profile(ctx, int(enable)), ctx)


def rgc_profile_read(ctx):
    ms = (C.c_float * RGC_NPHASE)()
    n = C.c_int(0)
    _check(lib().rgc_profile_read(ctx, ms, RGC_NPHASE, C.byref(n)), ctx)
    return dict(zip(PHASES, [float(x) for x in ms])), int(n.value)


def rgc_launch_count(ctx) -> int:
    return int(lib().rgc_launch_count(ctx))


# ----------------------------------------------------------- message blocks (host side)
def decode_block(blk, L: int, H: int):
    """One message block (include/rgc.h layout) -> [(idx uint32[], val float32[])] per layer.
    Plain layers' pairs come first, then the ASQ layers' indices; an ASQ layer's values
    are its header value word repeated."""
    import numpy as np
    blk = np.ascontiguousarray(blk, np.uint8)
    hdr = blk[:4 * H].view(np.uint32)
    words = blk[4 * H:4 * H + (blk.size - 4 * H) // 4 * 4].view(np.uint32)
    cnt = [int(hdr[l]) for l in range(L)]
    vw = [int(hdr[L + 2 + l]) for l in range(L)]
    plain = sum(c for c, v in zip(cnt, vw) if v == RGC_MSG_DENSE)
    po, qo = 0, 2 * plain
    out = []
    for l in range(L):
        c = cnt[l]
        if vw[l] == RGC_MSG_DENSE:
            pr = words[po:po + 2 * c].reshape(-1, 2)
            out.append((pr[:, 0].copy(), pr[:, 1].copy().view(np.float32)))
            po += 2 * c
        else:
            idx = words[qo:qo + c].copy()
            out.append((idx, np.full(c, vw[l], np.uint32).view(np.float32)))
            qo += c
    return out


def block_used_bytes(blk, L: int, H: int) -> int:
    import numpy as np
    hdr = np.ascontiguousarray(blk[:4 * H], np.uint8).view(np.uint32)
    return 4 * H + sum((8 if int(hdr[L + 2 + l]) == RGC_MSG_DENSE else 4) * int(hdr[l])
                       for l in range(L))


# ----------------------------------------------------------- convenience engine
@dataclass
class LayerSpec:
    n: int
    density: float = 0.001
    momentum: float = 0.0
    selector: int = RGC_SEL_TRIMMED
    bs_branch: int = RGC_BS_MONOTONE
    trim_eps: float = 0.0
    bs_eps: float = 0.0
    max_count: int = 0
    sample_interval: int = 0
    quantize: int = 0          # 1: ASQ, indices + one mean per message


@dataclass
class RGC:
    """One node's RGC state for a fixed list of compressed layers.

    torch provides the device memory (workspace, message, gathered buffer) and
    the stream; every step runs in librgc.so.  Residuals / momenta are the
    caller's tensors (V starts at 0)."""
    specs: list
    rank: int = 0
    nranks: int = 1
    device: int = 0
    uid: bytes | None = None
    sync_mode: int = RGC_SYNC_FIXED
    p2p_inspect: bool = False      # P2P / PULL: copy every rank's block into self.gathered
    prefill: bool = True           # step(): zero the outputs under the selection (prefill)
    ctx: object = field(default=None, init=False)

    def __post_init__(self):
        import torch
        self._torch = torch
        self.layers = make_layers(self.specs)
        self.L = len(self.specs)
        dev = torch.device("cuda", self.device)
        stream = torch.cuda.current_stream(dev).cuda_stream
        self.ctx = rgc_init(self.rank, self.nranks, self.device, self.uid, stream)
        self.sizes = rgc_sizes(self.ctx, self.layers)
        self.ws = torch.empty(self.sizes.workspace_bytes, dtype=torch.uint8, device=dev)
        if self.sync_mode in P2P_MODES:
            # the message block is library memory mapped by every peer (CUDA IPC);
            # self.gathered only receives inspection copies (p2p_inspect)
            self.msg = rgc_p2p_init(self.ctx, self.layers, self.sizes.msg_bytes)
            self.gathered = (torch.empty(self.sizes.gathered_bytes, dtype=torch.uint8, device=dev)
                             if self.p2p_inspect else None)
        else:
            self.msg = torch.empty(self.sizes.msg_bytes, dtype=torch.uint8, device=dev)
            if self.nranks == 1:
                self.gathered = self.msg
            else:
                self.gathered = torch.empty(self.sizes.gathered_bytes, dtype=torch.uint8, device=dev)
        rgc_workspace_init(self.ctx, self.layers, self.ws)

    def _stream(self):
        rgc_set_stream(self.ctx, self._torch.cuda.current_stream(self.device).cuda_stream)

    def compress(self, grads, residuals, momenta=None):
        self._stream()
        rgc_compress(self.ctx, self.layers, grads, residuals, momenta, self.msg, self.ws)

    def sync(self, mode=None, counts_host=None):
        self._stream()
        if self.sync_mode in P2P_MODES:
            rgc_sync(self.ctx, self.layers, self.msg, None, self.sync_mode, None)
            if self.p2p_inspect:
                rgc_p2p_gather(self.ctx, self.layers, self.gathered)
            return
        rgc_sync(self.ctx, self.layers, self.msg, self.gathered,
                 self.sync_mode if mode is None else mode, counts_host)

    def decompress(self, outs, ordered=True):
        self._stream()
        gathered = None if self.sync_mode in P2P_MODES else self.gathered
        rgc_decompress(self.ctx, self.layers, gathered, outs, self.ws, ordered)

    def prefill_outputs(self, outs):
        rgc_decompress_prefill(self.ctx, self.layers, outs)

    def step(self, grads, residuals, momenta, outs, ordered=True):
        """One iteration of compress -> sync -> decompress (asynchronous).  Raises RgcError
        when the context status (rgc_status, polled without a sync) reports an error of a
        step that has completed: a non-finite residual on any rank (RGC_ENONFINITE), an NCCL
        async error (RGC_ENCCL) or a timed-out cross-GPU wait (RGC_ESTATE)."""
        if self.prefill:
            self.prefill_outputs(outs)
        self.compress(grads, residuals, momenta)
        try:
            self.sync()
        except RgcError as e:
            # RGC_SYNC_SIZES_FIRST reports a non-finite residual after completing the
            # exchange: finish the step (the context stays consistent), then raise
            if e.code != RGC_ENONFINITE:
                raise
            self.decompress(outs, ordered)
            raise
        self.decompress(outs, ordered)
        rgc_status(self.ctx, 0)

    def check(self, clear=False):
        """Wait for the enqueued work and raise RgcError if any completed step reported an
        error (clear=True resets a non-finite report afterwards)."""
        rgc_status(self.ctx, RGC_STATUS_CLEAR if clear else RGC_STATUS_WAIT)

    def status(self, wait=True):
        """(rc, words) of rgc_status without raising."""
        return rgc_status(self.ctx, RGC_STATUS_WAIT if wait else 0, raise_on_error=False)

    def info(self):
        return rgc_get_info(self.ctx, self.L, self.ws)

    # measurement helpers (the same names on RGCBuckets)
    def launch_count(self):
        return rgc_launch_count(self.ctx)

    def profile(self, mode):
        rgc_profile(self.ctx, mode)

    def profile_read(self):
        return rgc_profile_read(self.ctx)

    def message_bytes(self, counts):
        """Bytes of a message with these per-layer counts (header + 8 per pair, 4 per ASQ index)."""
        return 4 * self.header_words() + sum((4 if s.quantize else 8) * int(c)
                                             for s, c in zip(self.specs, counts))

    def header_words(self):
        return int(self.sizes.header_bytes // 4)

    def messages(self, gathered=None):
        """Host view of every rank's message: list over ranks of list over layers of
        (idx uint32[], val float32[]) -- a device->host read for tests / stats.  An
        ASQ layer's values are its single quantized value repeated."""
        g = (self.gathered if gathered is None else gathered).cpu().numpy()
        stride = int(self.sizes.msg_bytes)
        return [decode_block(g[r * stride:(r + 1) * stride], self.L, self.header_words())
                for r in range(g.size // stride)]

    def used_bytes(self, gathered=None, rank=0):
        """Bytes of rank `rank`'s block that carry data (header + pairs + ASQ indices)."""
        g = (self.gathered if gathered is None else gathered).cpu().numpy()
        stride = int(self.sizes.msg_bytes)
        return block_used_bytes(g[rank * stride:(rank + 1) * stride], self.L, self.header_words())

    def close(self):
        if self.ctx is not None:
            rgc_finalize(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class RGCBuckets:
    """A step split into buckets of layers (NEXT-3 bucketing; P:383-406 overlaps the
    synchronisation of finished layers with the remaining computation): one RGC context per
    bucket, each on its own CUDA stream, forked from and joined back to the caller's stream
    every step, so one bucket's latency-bound selection chain runs while another bucket's
    accumulate pass (K1) streams.  Results are those of one RGC over all layers (the layers
    are independent); the exchange carries one message per bucket.

    groups: lists of layer indices (a partition of range(len(specs))), in launch order.
    k1_occ: per bucket, K1's CTAs per SM (None: the occupancy limit) -- a bucket whose K1 runs
      beside another bucket's selection leaves room for it (RGC_K1_OCC).
    priority: per bucket stream priority (lower = higher priority, torch convention).
    uids: per bucket NCCL unique id (nranks > 1: one communicator per context)."""

    def __init__(self, specs, groups, rank=0, nranks=1, device=0, uids=None,
                 sync_mode=RGC_SYNC_FIXED, k1_occ=None, priority=None, prefill=True):
        import torch
        self._torch = torch
        self.specs = specs
        self.groups = [list(g) for g in groups]
        assert sorted(i for g in self.groups for i in g) == list(range(len(specs)))
        self.device = device
        self.L = len(specs)
        self.engs, self.streams = [], []
        for b, g in enumerate(self.groups):
            occ = (k1_occ or [None] * len(groups))[b]
            if occ:
                os.environ["RGC_K1_OCC"] = str(occ)
            try:
                self.engs.append(RGC([specs[i] for i in g], rank=rank, nranks=nranks,
                                     device=device, uid=(uids or [None] * len(groups))[b],
                                     sync_mode=sync_mode, prefill=prefill))
            finally:
                os.environ.pop("RGC_K1_OCC", None)
            pr = (priority or [0] * len(groups))[b]
            self.streams.append(torch.cuda.Stream(device=device, priority=pr))
        self.ctx = self.engs[0].ctx
        from types import SimpleNamespace
        self.sizes = SimpleNamespace(msg_bytes=sum(int(e.sizes.msg_bytes) for e in self.engs),
                                     k_total=sum(int(e.sizes.k_total) for e in self.engs),
                                     workspace_bytes=sum(int(e.sizes.workspace_bytes) for e in self.engs))

    def step(self, grads, residuals, momenta, outs, ordered=True):
        torch = self._torch
        cur = torch.cuda.current_stream(self.device)
        for st in self.streams:
            st.wait_stream(cur)
        for eng, st, g in zip(self.engs, self.streams, self.groups):
            with torch.cuda.stream(st):
                eng.step([grads[i] for i in g], [residuals[i] for i in g],
                         None if momenta is None else [momenta[i] for i in g],
                         [outs[i] for i in g], ordered)
        for st in self.streams:
            cur.wait_stream(st)

    def info(self):
        out = [None] * self.L
        for eng, g in zip(self.engs, self.groups):
            for i, x in zip(g, eng.info()):
                out[i] = x
        return out

    def launch_count(self):
        return sum(e.launch_count() for e in self.engs)

    def profile(self, mode):
        for e in self.engs:
            e.profile(mode)

    def profile_read(self):
        """Per-phase milliseconds summed over the buckets (the buckets overlap: not a
        critical path) and the per-bucket dicts."""
        per = [e.profile_read() for e in self.engs]
        tot = {k: sum(p[0][k] for p in per) for k in PHASES}
        return tot, per[0][1], [p[0] for p in per]

    def message_bytes(self, counts):
        return sum(e.message_bytes([counts[i] for i in g]) for e, g in zip(self.engs, self.groups))

    def status(self, wait=True):
        res = [e.status(wait) for e in self.engs]
        return max(r[0] for r in res), [r[1] for r in res]

    def check(self, clear=False):
        for e in self.engs:
            e.check(clear)

    def close(self):
        for e in self.engs:
            e.close()
