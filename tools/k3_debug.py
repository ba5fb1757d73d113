import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import oracle as O, synth
from harness import spec, bits
from paper_1808_04357_b200 import rgc as R
for sel in (0, 1):
  for n in (65537, 4097, 1000000):
    s = spec(n, sel=sel)
    eng = R.RGC([s], nranks=1, device=0)
    dev = torch.device("cuda", 0)
    V = [torch.zeros(n, device=dev)]; U = [torch.zeros(n, device=dev)]
    Vo = np.zeros(n, np.float32); Uo = np.zeros(n, np.float32)
    for it in range(3):
        g = synth.gradient(n, "gaussian", seed=0, rank=0, layer=0, it=it)
        eng.compress([torch.from_numpy(g).to(dev)], V, U)
        torch.cuda.synchronize()
        info = eng.info()[0]
        (gi, gv), = eng.messages(eng.msg)[0]
        idx, val, oi = O.compress_layer(g, Uo, Vo, s.momentum, s.density, s.selector)
        ok = np.array_equal(gi, idx) and np.array_equal(bits(gv), bits(val))
        print(f"sel={sel} n={n} it={it} ok={ok} count gpu={info['count']} emitted={info['emitted']} oracle={len(idx)} surv gpu={info['survivors']} oracle={oi['survivors']} flags={hex(info['flags'])}/{hex(oi['flags'])} maxidx={gi.max() if len(gi) else -1}", flush=True)
        if not ok:
            bad = np.nonzero((gi[:min(len(gi),len(idx))] != idx[:min(len(gi),len(idx))]))[0]
            print("  first bad", bad[:10], gi[bad[:5]] if len(bad) else None, idx[bad[:5]] if len(bad) else None)
            Vg = V[0].cpu().numpy(); print("  residual equal:", np.array_equal(bits(Vg), bits(Vo)))
            break
    eng.close()
