"""Host time per API call of an eager step (which call blocks?)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_1808_04357_b200 import rgc as R

sizes, kinds = synth.model_layers("vgg16")
specs = [R.LayerSpec(n=n, density=0.001, momentum=0.9, selector=synth.selector_for("vgg16", k, "hybrid"))
         for n, k in zip(sizes, kinds)]
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev); gen.manual_seed(1)
NS = int(os.environ.get("NSETS", "8"))
G = [[torch.randn(n, device=dev, generator=gen) * 0.01 for n in sizes] for _ in range(NS)]
V = [torch.zeros(n, device=dev) for n in sizes]
U = [torch.zeros(n, device=dev) for n in sizes]
O = [torch.empty(n, device=dev) for n in sizes]
eng = R.RGC(specs, device=0, prefill=True)
acc = [0.0] * 4
for i in range(40):
    t = [time.perf_counter()]
    eng.prefill_outputs(O); t.append(time.perf_counter())
    eng.compress(G[i % NS], V, U); t.append(time.perf_counter())
    eng.sync(); t.append(time.perf_counter())
    eng.decompress(O); t.append(time.perf_counter())
    if i >= 10:
        for j in range(4):
            acc[j] += t[j + 1] - t[j]
print(f"NSETS={NS} host ms per call (prefill, compress, sync, decompress):",
      [round(a * 1e3 / 30, 3) for a in acc], flush=True)
