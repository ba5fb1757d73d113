import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O, synth
from paper_1808_04357_b200 import rgc as R
dev = torch.device("cuda", 0)
for n, sel in [(31, 1), (4095, 1), (31, 0)]:
    specs = [R.LayerSpec(n=n, density=0.001, momentum=0.9, selector=sel)]
    e = R.RGC(specs)
    g = synth.gradient(n, "gaussian", seed=0, rank=0, layer=0, it=0)
    V = [torch.zeros(n, device=dev)]; U = [torch.zeros(n, device=dev)]
    e.compress([torch.from_numpy(g).to(dev)], V, U)
    torch.cuda.synchronize()
    info = e.info()[0]
    msgs = e.messages(e.msg)[0][0]
    Vo = np.zeros(n, np.float32); Uo = np.zeros(n, np.float32)
    idx, val, oi = O.compress_layer(g, Uo, Vo, 0.9, 0.001, sel)
    print("n", n, "sel", sel, "gpu count", info["count"], "emitted", info["emitted"], "thr", info["threshold"], "flags", hex(info["flags"]))
    print("  oracle idx", idx[:10], "thr", oi["threshold"], "count", oi["count"])
    print("  gpu idx", msgs[0][:10], msgs[1][:10])
    hdr = e.msg[:64].cpu().numpy().view(np.uint32)
    print("  hdr", hdr[:8])
    a = np.abs(g)
    print("  top |g|", np.sort(a)[::-1][:5], "n>thr", (a > np.float32(oi["threshold"])).sum())
    Vg = V[0].cpu().numpy()
    print("  V zero count gpu", (Vg == 0).sum(), "oracle", (Vo == 0).sum())
    e.close()
