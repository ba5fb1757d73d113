"""The launch-shape choices the library makes from the layer list, forced both ways, against
the oracle (each configuration in its own process: the knobs are read once per process).

* K45 cluster size (rgc_api.cu make_layout): 4-CTA clusters, or 2-CTA clusters when the
  K45-capable layers need more than one wave -- RGC_K45_CL = 2 / 4 forces either on a list
  where the default would pick the other (sets between the two capacities take K4 + K3B).
* K2's V passes inside the stash launch (small lists) or as their own launches:
  RGC_FOLD_K2_TILES = 0 / a large value.
* The one-launch K4 (cooperative, grid barriers) or three launches: RGC_NO_COOP_K4.
* K3A over the candidate stash: one K1 record per segment, or several small records grouped
  (one flat index through their counts): RGC_K3A_SEGREC = 1 / 5.

Bit-exact selection, residuals and decompression through harness.run, several iterations so
the candidate stash serves K2 / K3 and the finalisations see warm state.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r"""
import sys
sys.path.insert(0, {tests!r})
sys.path.insert(0, {root!r})
from harness import run, spec
# many Alg.2 layers (more K45-capable layers than one wave of 4-CTA clusters), a large Alg.2
# layer whose survivors exceed the 2-CTA capacity, Alg.3 / sampled layers and a tiny one
specs = [spec(20_000 + 977 * i, sel=0) for i in range(40)]
specs += [spec(12_000_000, sel=0), spec(1_500_001, sel=1), spec(300_007, sel=2, interval=3),
          spec(4097, sel=0, m=0.0)]
run(specs, p=2, iters=4, dist="t3", seed=11, where={tag!r})
run(specs[:6], p=1, iters=3, dist="gaussian", seed=12, where={tag!r} + " small")
print("ok")
"""

CONFIGS = {
    "k45_cl2": {"RGC_K45_CL": "2"},
    "k45_cl4": {"RGC_K45_CL": "4"},
    "fold_all": {"RGC_FOLD_K2_TILES": "100000000"},
    "fold_none": {"RGC_FOLD_K2_TILES": "0"},
    "k4_three_launches": {"RGC_NO_COOP_K4": "1"},
    "k3a_records_1": {"RGC_K3A_SEGREC": "1"},
    "k3a_records_5": {"RGC_K3A_SEGREC": "5"},
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_forced_launch_shapes(name):
    env = dict(os.environ)
    env.update(CONFIGS[name])
    code = CASE.format(tests=os.path.join(ROOT, "tests"), root=ROOT, tag=name)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (name, r.stdout[-2000:],
                                                                    r.stderr[-4000:])


ALIAS = r"""
import sys
sys.path.insert(0, {tests!r})
sys.path.insert(0, {root!r})
import numpy as np, torch
import oracle as O, synth
from harness import bits, spec
from paper_1808_04357_b200 import rgc as R
# include/rgc.h: the prefill outputs may alias the gradients -- the fill must then not start
# before K1 has read them, whatever the fill placement (RGC_FILL_AT)
specs = [spec(300_001, sel=0), spec(1_000_003, sel=1), spec(65_537, sel=0, m=0.0)]
dev = torch.device("cuda", 0)
eng = R.RGC(specs, device=0)
assert eng.prefill
V = [torch.zeros(s.n, device=dev) for s in specs]
U = [torch.zeros(s.n, device=dev) for s in specs]
Vo = [np.zeros(s.n, np.float32) for s in specs]
Uo = [np.zeros(s.n, np.float32) for s in specs]
for it in range(4):
    g = [synth.gradient(s.n, "gaussian", seed=5, layer=l, it=it) for l, s in enumerate(specs)]
    G = [torch.from_numpy(x).to(dev) for x in g]
    eng.step(G, V, U, G)            # out[l] is grad[l]
    torch.cuda.synchronize()
    for l, s in enumerate(specs):
        idx, val, oi = O.compress_layer(g[l], Uo[l], Vo[l], s.momentum, s.density, s.selector,
                                        s.bs_branch, 0.2, 1e-3, 0)
        want = O.decompress(s.n, [(idx, val)])
        assert np.array_equal(bits(G[l].cpu().numpy()), bits(want)), (it, l, "decompress")
        assert np.array_equal(bits(V[l].cpu().numpy()), bits(Vo[l])), (it, l, "residual")
eng.check()
eng.close()
print("ok")
"""


@pytest.mark.parametrize("fill_at", ["0", "1", "default"])
def test_prefill_outputs_aliasing_gradients(fill_at):
    env = dict(os.environ)
    if fill_at != "default":
        env["RGC_FILL_AT"] = fill_at
    code = ALIAS.format(tests=os.path.join(ROOT, "tests"), root=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), (fill_at, r.stdout[-2000:],
                                                                    r.stderr[-4000:])
