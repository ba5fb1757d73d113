"""Eager step timing variants (prefill on/off, default vs side torch stream)."""
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

def run(prefill, side, steps=30):
    V = [torch.zeros(n, device=dev) for n in sizes]
    U = [torch.zeros(n, device=dev) for n in sizes]
    O = [torch.empty(n, device=dev) for n in sizes]
    eng = R.RGC(specs, device=0, prefill=prefill)
    s = torch.cuda.Stream() if side else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        for i in range(8):
            eng.step(G[i % NS], V, U, O)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        for i in range(steps):
            eng.step(G[i % NS], V, U, O)
        e1.record(s)
        th = time.perf_counter() - t0
        torch.cuda.synchronize()
    eng.close()
    print(f"NSETS={NS} prefill={prefill} side={side} inline={os.environ.get('RGC_FILL_INLINE')}: "
          f"{e0.elapsed_time(e1)/steps:.3f} ms/step (host enqueue {th*1e3/steps:.3f} ms/step)", flush=True)

for pf in (False, True):
    run(pf, False)
