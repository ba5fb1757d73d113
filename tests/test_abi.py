"""The C-ABI boundary on CPU: the library loads, exports every symbol include/rgc.h
declares, and its host-side logic (k, validation, buffer sizes) is right.
No compute calls (there is no GPU here)."""
import os
import re
import subprocess
import sys

import pytest

import oracle as O
from paper_1808_04357_b200 import rgc as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    txt = open(os.path.join(ROOT, "include", "rgc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rgc_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = R.lib()
    names = declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", R.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r" T (rgc_\w+)", out))
    assert set(names) <= exported


def test_version_and_k_match_oracle():
    assert "sm_100a" in R.rgc_version()
    for n in [1, 7, 999, 1000, 1001, 4096, 1_000_000, 102_760_448, 2**31 - 1]:
        for D in [0.001, 0.01, 0.1, 1 / 64, 0.25, 1.0]:
            assert R.rgc_k(n, D) == O.k_of(n, D)


def sizes(specs):
    return R.rgc_sizes(None, R.make_layers(specs))


@pytest.mark.parametrize("bad", [
    dict(n=0), dict(n=2**31), dict(n=100, density=0.0), dict(n=100, density=1.5),
    dict(n=100, momentum=-1.0), dict(n=100, selector=3), dict(n=100, bs_branch=3),
    dict(n=100, bs_eps=1e-4), dict(n=100, bs_eps=1.0), dict(n=100, trim_eps=0.01),
    dict(n=100, trim_eps=1.5), dict(n=100_000, density=0.01, max_count=5),
])
def test_validation_rejects(bad):
    with pytest.raises(R.RgcError) as e:
        sizes([R.LayerSpec(**bad)])
    assert e.value.code == R.RGC_EINVAL


def test_layer_count_limits():
    with pytest.raises(R.RgcError):
        sizes([R.LayerSpec(n=10)] * 129)
    assert sizes([R.LayerSpec(n=10)] * 128).k_total == 128


def test_buffer_sizes_arithmetic():
    specs = [R.LayerSpec(n=1_000_000, selector=0), R.LayerSpec(n=1_000_000, selector=1),
             R.LayerSpec(n=999, selector=1, max_count=50), R.LayerSpec(n=5, density=1.0)]
    s = sizes(specs)
    k = [1000, 1000, 1, 5]
    cap = [1000, 2000, 50, 5]
    assert s.k_total == sum(k)
    assert s.cap_total == sum(cap)
    H = 4 * ((2 * len(specs) + 3 + 3) // 4)     # counts, status, L, value words, table marker

    def tab_bytes(ns):   # the producer's range table: one word per 8192-tile boundary per layer
        return 4 * ((sum((n + 8191) // 8192 for n in ns) + len(ns) + 3) // 4 * 4)
    assert s.header_bytes == 4 * H
    assert s.msg_bytes == (4 * H + 8 * sum(cap) + 15) // 16 * 16 + tab_bytes([1_000_000, 1_000_000, 999, 5])
    # ASQ layers need 4 bytes per entry (index only)
    q = sizes([R.LayerSpec(n=1_000_000, selector=0, quantize=1),
               R.LayerSpec(n=1_000_000, selector=1, quantize=1), R.LayerSpec(n=5, density=1.0)])
    Hq = 4 * ((2 * 3 + 3 + 3) // 4)
    assert q.msg_bytes == (4 * Hq + 4 * (1000 + 2000) + 8 * 5 + 15) // 16 * 16 + tab_bytes([1_000_000, 1_000_000, 5])
    with pytest.raises(R.RgcError):   # sampled BS cannot be used with quantization
        sizes([R.LayerSpec(n=1000, selector=2, quantize=1)])
    assert s.gathered_bytes == s.msg_bytes
    assert s.workspace_bytes > 0


def test_product_never_imports_oracle_and_vice_versa():
    pkg = os.path.join(ROOT, "paper_1808_04357_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "rgc_oracle" not in txt and "rgco_" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"(import|from)\s+paper_1808_04357_b200", txt), f
            assert "#include" not in txt or "rgc.h" not in txt, f
            assert "librgc.so" not in txt, f


def test_missing_library_fails_loudly(tmp_path):
    code = ("import paper_1808_04357_b200.rgc as R\n"
            "R.LIB_PATH = '/nonexistent/librgc.so'\nR._lib = None\n"
            "try:\n    R.lib()\nexcept ImportError as e:\n    print('LOUD', e)\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert "LOUD" in out.stdout
