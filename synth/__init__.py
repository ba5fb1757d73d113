"""Seeded synthetic inputs shared by the oracle-side tests, the CUDA-side tests
and bench.py.  Holds NONE of the method's arithmetic: only random numbers and
the per-layer tensor sizes of the paper's workloads.

Recipe: every gradient tensor is drawn from a
``torch.Generator`` on the CPU seeded with a hash of
(seed, rank, layer, iteration), so different ranks hold different gradients
("very few overlapping indices"), and the same host arrays feed both
the oracle and the GPU path.
"""
from __future__ import annotations

import hashlib

import numpy as np
import torch

# ---- per-layer sizes of the compressed tensors (4·n > 131072 B) ----
# torchvision 0.26 shapes; LSTMs: 2x1500 tied LM.
VGG16 = ([36_864, 73_728, 147_456, 294_912, 589_824, 589_824, 1_179_648]
         + [2_359_296] * 5 + [102_760_448, 16_777_216, 4_096_000])
VGG16_KIND = ["conv"] * 12 + ["fc"] * 3
ALEXNET = [307_200, 663_552, 884_736, 589_824, 37_748_736, 16_777_216, 4_096_000]
ALEXNET_KIND = ["conv"] * 4 + ["fc"] * 3
RESNET50 = ([36_864] * 3 + [65_536] * 7 + [131_072] * 2 + [147_456] * 4
            + [262_144] * 11 + [524_288] * 2 + [589_824] * 6 + [1_048_576] * 5
            + [2_048_000] + [2_097_152] + [2_359_296] * 3)
RESNET50_KIND = ["conv"] * 44 + ["fc"]
LSTM_PTB = [15_000_000] + [9_000_000] * 4
LSTM_PTB_KIND = ["embed"] + ["hidden"] * 4
LSTM_WIKI2 = [49_917_000] + [9_000_000] * 4 + [33_278]
LSTM_WIKI2_KIND = ["embed"] + ["hidden"] * 4 + ["softmax_bias"]

# elements of the tensors each model leaves UNcompressed (4·n <= 131072 B): the paper
# synchronises them with a dense allreduce; SURVEY 8(d) totals minus the compressed sizes
SMALL_ELEMENTS = {"vgg16": 15_144, "alexnet": 33_576, "resnet50": 198_696, "lstm_ptb": 34_000,
                  "lstm_wiki2": 24_000, "c1": 0, "m1": 0}

MODELS = {
    "vgg16": (VGG16, VGG16_KIND),
    "alexnet": (ALEXNET, ALEXNET_KIND),
    "resnet50": (RESNET50, RESNET50_KIND),
    "lstm_ptb": (LSTM_PTB, LSTM_PTB_KIND),
    "lstm_wiki2": (LSTM_WIKI2, LSTM_WIKI2_KIND),
    "c1": ([1_000_000], ["fc"]),
    "m1": ([100_000_000], ["fc"]),
}

DISTS = ("gaussian", "uniform", "laplace", "t3", "cauchy", "sparse", "equal", "zero",
         "subnormal", "ties")


def seed_of(*parts) -> int:
    h = hashlib.sha256(repr(tuple(parts)).encode()).digest()
    return int.from_bytes(h[:8], "little") & ((1 << 63) - 1)


def gradient(n: int, dist: str = "gaussian", *, seed: int = 0, rank: int = 0,
             layer: int = 0, it: int = 0, scale: float = 0.01) -> np.ndarray:
    """One synthetic fp32 gradient tensor of n elements (host, C-contiguous)."""
    gen = torch.Generator(device="cpu")
    gen.manual_seed(seed_of(seed, rank, layer, it, dist))
    if n == 0:
        return np.zeros(0, np.float32)
    if dist == "gaussian":
        x = torch.randn(n, generator=gen, dtype=torch.float32) * scale
    elif dist == "uniform":           # Fig. 3's "standard uniform" data
        x = torch.rand(n, generator=gen, dtype=torch.float32)
    elif dist == "laplace":
        u = torch.rand(n, generator=gen, dtype=torch.float64) - 0.5
        x = (-torch.sign(u) * torch.log1p(-2 * u.abs()) * scale).float()
    elif dist == "t3":                # Student-t, nu = 3 (heavy tailed, C4)
        z = torch.randn(n, generator=gen, dtype=torch.float64)
        c = torch.randn(n, 3, generator=gen, dtype=torch.float64).pow(2).sum(1)
        x = (z / torch.sqrt(c / 3.0) * scale).float()
    elif dist == "cauchy":
        u = torch.rand(n, generator=gen, dtype=torch.float64)
        x = (torch.tan(np.pi * (u - 0.5)) * scale).float()
    elif dist == "sparse":            # 99 % exact zeros
        x = torch.randn(n, generator=gen, dtype=torch.float32) * scale
        keep = torch.rand(n, generator=gen) < 0.01
        x = torch.where(keep, x, torch.zeros_like(x))
    elif dist == "equal":             # all-equal magnitudes, random signs
        s = torch.randint(0, 2, (n,), generator=gen).float() * 2 - 1
        x = s * scale
    elif dist == "zero":
        x = torch.zeros(n, dtype=torch.float32)
    elif dist == "subnormal":         # magnitudes spread over subnormals / tiny normals
        e = torch.randint(-149, -120, (n,), generator=gen).double()
        s = torch.randint(0, 2, (n,), generator=gen).double() * 2 - 1
        m = torch.rand(n, generator=gen, dtype=torch.float64) + 1.0
        x = (s * m * torch.pow(2.0, e)).float()
    elif dist == "ties":              # few distinct magnitudes -> many exact ties
        v = torch.randint(-4, 5, (n,), generator=gen).float() * scale
        x = v
    else:
        raise ValueError(dist)
    return np.ascontiguousarray(x.numpy(), dtype=np.float32)


def model_layers(model: str):
    sizes, kinds = MODELS[model]
    return list(sizes), list(kinds)


def selector_for(model: str, kind: str, policy: str = "hybrid") -> int:
    """Per-layer selector (A11): 0 trimmed, 1 threshold BS.

    hybrid: trimmed for conv layers, threshold binary search for LSTM hidden /
    embedding-softmax layers and for CNN fully-connected layers (P:195-196
    names VGG16 fc6 as a threshold-search case)."""
    if policy == "trimmed":
        return 0
    if policy == "bs":
        return 1
    return 0 if kind == "conv" else 1
