"""N > 1 path.

CPU (gloo, world_size 2): the message block contract (header of length
elements + compact ascending pairs), both exchange schemes of
rgc_sync (fixed-capacity allgather; sizes first then exact-size broadcasts,
planned by the library's host-side rgc_sync_plan) and rank-ordered
decompression, with oracle-built messages; AGREEMENT across ranks and equality
with a single-process simulation of all ranks.

GPU (NCCL, torchrun): tests/mgpu_worker.py on 2 (and 4) GPUs through the C ABI.
"""
import hashlib
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as O
import synth
from paper_1808_04357_b200 import rgc as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPECS = [dict(n=70_001, density=0.001, momentum=0.9, selector=0),
         dict(n=33_333, density=0.003, momentum=0.9, selector=1),
         dict(n=5_000, density=0.01, momentum=0.0, selector=1, bs_branch=1),
         dict(n=40_000, density=0.002, momentum=0.9, selector=0, quantize=1),
         dict(n=20_011, density=0.004, momentum=0.0, selector=1, quantize=1)]


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


DENSE = 0xFFFFFFFF   # header value word of a plain layer (include/rgc.h)


def pack_block(msgs, L, H, msg_bytes, status=0):
    """msgs[l] = (idx, val) for a plain layer or (idx, qmean float) for an ASQ layer.
    Layout (include/rgc.h): counts, status, L, value words; plain pairs, then ASQ indices."""
    blk = np.zeros(msg_bytes, np.uint8)
    hdr = blk[:4 * H].view(np.uint32)
    words = blk[4 * H:4 * H + (msg_bytes - 4 * H) // 4 * 4].view(np.uint32)
    o = 0
    for l, (idx, val) in enumerate(msgs):
        hdr[l] = len(idx)
        if isinstance(val, np.ndarray):
            hdr[L + 2 + l] = DENSE
            words[o:o + 2 * len(idx):2] = idx
            words[o + 1:o + 2 * len(idx):2] = val.view(np.uint32)
            o += 2 * len(idx)
    for l, (idx, val) in enumerate(msgs):
        if not isinstance(val, np.ndarray):
            hdr[L + 2 + l] = np.float32(val).view(np.uint32)
            words[o:o + len(idx)] = idx
            o += len(idx)
    hdr[L] = status
    hdr[L + 1] = L
    return blk


def unpack_block(blk, L, H):
    """-> [(idx, val)] with an ASQ layer's value repeated over its indices."""
    hdr = blk[:4 * H].view(np.uint32)
    words = blk[4 * H:4 * H + (blk.size - 4 * H) // 4 * 4].view(np.uint32)
    out, o = [None] * L, 0
    for l in range(L):
        c = int(hdr[l])
        if hdr[L + 2 + l] == DENSE:
            out[l] = (words[o:o + 2 * c:2].copy(), words[o + 1:o + 2 * c:2].copy().view(np.float32))
            o += 2 * c
    for l in range(L):
        c = int(hdr[l])
        if hdr[L + 2 + l] != DENSE:
            out[l] = (words[o:o + c].copy(), np.full(c, hdr[L + 2 + l], np.uint32).view(np.float32))
            o += c
    return out


def used_bytes(blk, L, H):
    hdr = blk[:4 * H].view(np.uint32)
    return 4 * H + sum((8 if hdr[L + 2 + l] == DENSE else 4) * int(hdr[l]) for l in range(L))


def oracle_rank_messages(rank, it, state):
    msgs = []
    for l, s in enumerate(SPECS):
        g = synth.gradient(s["n"], "gaussian", seed=3, rank=rank, layer=l, it=it)
        V, u, asq = state[l]
        idx, val, info = O.compress_layer(g, u, V, s["momentum"], s["density"], s["selector"],
                                          s.get("bs_branch", 0), asq=asq)
        msgs.append((idx, val) if asq is None else (idx, np.float32(info["qmean"])))
    return msgs


def new_state():
    return [(np.zeros(s["n"], np.float32),
             np.zeros(s["n"], np.float32) if s["momentum"] else None,
             O.AsqState() if s.get("quantize") else None) for s in SPECS]


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = len(SPECS)
    sz = R.rgc_sizes(None, R.make_layers(SPECS))
    H, MB = int(sz.header_bytes // 4), int(sz.msg_bytes)
    state = new_state()
    results = []
    for it in range(2):
        blk = pack_block(oracle_rank_messages(rank, it, state), L, H, MB)
        # RGC_SYNC_FIXED: one allgather of the fixed-capacity block
        outl = [torch.zeros(MB, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(outl, torch.from_numpy(blk))
        fixed = [t.numpy() for t in outl]
        # RGC_SYNC_SIZES_FIRST: headers, host plan, exact-size broadcasts
        hl = [torch.zeros(4 * H, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(hl, torch.from_numpy(blk[:4 * H].copy()))
        headers = np.concatenate([t.numpy().view(np.uint32) for t in hl])
        nbytes, counts, status = R.rgc_sync_plan(headers, world, L, H, MB)
        sizes_first = []
        for r in range(world):
            buf = torch.from_numpy(blk[:int(nbytes[r])].copy()) if r == rank else \
                torch.zeros(int(nbytes[r]), dtype=torch.uint8)
            dist.broadcast(buf, src=r)
            full = np.zeros(MB, np.uint8)
            full[:int(nbytes[r])] = buf.numpy()
            sizes_first.append(full)
        dec_f = [unpack_block(b, L, H) for b in fixed]
        dec_s = [unpack_block(b, L, H) for b in sizes_first]
        outs = []
        for l, s in enumerate(SPECS):
            a = O.decompress(s["n"], [dec_f[r][l] for r in range(world)])
            b = O.decompress(s["n"], [dec_s[r][l] for r in range(world)])
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
            outs.append(a)
        want_bytes = [used_bytes(b, L, H) for b in fixed]
        assert [int(x) for x in nbytes] == want_bytes and status == 0
        assert [int(x) for x in counts] == [len(dec_f[r][l][0]) for r in range(world) for l in range(L)]
        h = hashlib.sha256(b"".join(o.tobytes() for o in outs)).hexdigest()
        results.append((h, [o.copy() for o in outs]))
    digests = [None] * world
    dist.all_gather_object(digests, [r[0] for r in results])
    dist.destroy_process_group()
    q.put((rank, digests, [r[1] for r in results]))


def test_gloo_two_ranks_sync_contract():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    got.sort(key=lambda x: x[0])
    digests = got[0][1]                  # [rank][iteration] digest of the decompressed output
    assert digests == got[1][1]
    assert digests[0] == digests[1]      # AGREEMENT across ranks
    # single-process simulation of both ranks
    states = [new_state(), new_state()]
    for it in range(2):
        msgs = [oracle_rank_messages(r, it, states[r]) for r in range(2)]
        for l, s in enumerate(SPECS):
            want = O.decompress(s["n"], [(msgs[r][l][0], np.broadcast_to(
                np.float32(msgs[r][l][1]), msgs[r][l][0].shape)) for r in range(2)])
            assert np.array_equal(got[0][2][it][l].view(np.uint32), want.view(np.uint32))


def test_sync_plan_rejects_inconsistent_headers():
    H = 8
    hdr = np.zeros(2 * H, np.uint32)
    hdr[[0, 1, 2]] = [3, 4, 0]
    hdr[4] = 3                         # hdr[L+1] = L
    hdr[5:8] = DENSE                   # plain layers
    hdr[H:H + 3] = [1, 1, 1]
    hdr[H + 4] = 2                     # wrong L on rank 1
    hdr[H + 5:H + 8] = [DENSE, 0x3F800000, DENSE]   # rank 1: layer 1 is ASQ (4 B/entry)
    with pytest.raises(R.RgcError):
        R.rgc_sync_plan(hdr, 2, 3, H, 4096)
    hdr[H + 4] = 3
    b, c, st = R.rgc_sync_plan(hdr, 2, 3, H, 4096)
    assert list(b) == [4 * H + 8 * 7, 4 * H + 8 + 4 + 8] and list(c) == [3, 4, 0, 1, 1, 1]
    with pytest.raises(R.RgcError):   # header too short for the value words
        R.rgc_sync_plan(hdr, 2, 3, 7, 4096)
    hdr[0] = 10_000                    # exceeds capacity
    with pytest.raises(R.RgcError):
        R.rgc_sync_plan(hdr, 2, 3, H, 4096)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4])
def test_nccl_multi_gpu_parity(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    log = os.path.join(ROOT, "gpurun_out", f"mgpu_worker_n{n}.log")
    try:
        os.makedirs(os.path.dirname(log), exist_ok=True)
        with open(log, "w") as f:
            f.write(out.stdout + "\n---- stderr ----\n" + out.stderr)
    except OSError:
        pass
    assert "MGPU_RESULT OK" in out.stdout, out.stdout[-4000:] + out.stderr[-4000:]
