import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch
from harness import Sim, spec, grads_for
specs = [spec(1_000_000, sel=2, interval=5, m=0.9), spec(300_007, sel=2, interval=3, m=0.0)]
sim = Sim(specs, p=1)
for it in range(12):
    try:
        sim.step(grads_for(specs, 1, "gaussian", 5, it), where=f"it={it}")
        print("it", it, [ (hex(i["flags"]), i["count"]) for i in sim.eng[0].info()], flush=True)
    except Exception as e:
        print("FAIL it", it, repr(e)[:300]); break
