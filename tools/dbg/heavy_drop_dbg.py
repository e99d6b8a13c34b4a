import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from oracle import moe_oracle as O
from paper_2201_05596_b200 import arch as A
from paper_2201_05596_b200.gating import GatingConfig
S, M, E = 65536, 2048, 128
spec = A.LayerSpec(kind="moe", hidden=M, experts=E, gating=GatingConfig(E, 1, 1.0))
dev = "cuda"
gen = torch.Generator(device=dev).manual_seed(7)
gw = torch.randn(M, E, device=dev, generator=gen) * M ** -0.5
gw[0] = torch.randn(E, device=dev, generator=gen) * 0.5
gw = gw.to(torch.bfloat16)
w1 = torch.randn(E, M, 4 * M, device=dev, generator=gen, dtype=torch.bfloat16) * 0.1
w2 = torch.randn(E, 4 * M, M, device=dev, generator=gen, dtype=torch.bfloat16) * 0.1
b1 = torch.randn(E, 1, 4 * M, device=dev, generator=gen) * 0.05
b2 = torch.randn(E, 1, M, device=dev, generator=gen) * 0.05
p = A.MoeLayerParams(gate_w=gw, experts=tuple(A.FfnParams(w1[e], b1[e], w2[e], b2[e]) for e in range(E)))
x = torch.randn(S, M, device=dev, generator=gen).to(torch.bfloat16)
x[:, 0] = 1.0
outs = {}
for fuse in (True, False):
    layer = A.MoeLayer(spec, p, dtype=torch.bfloat16, fuse_combine=fuse)
    logits = torch.empty(S, E, device=dev)
    outs[fuse] = layer(x, logits_out=logits).clone()
    torch.cuda.synchronize()
ids, gp, slots, load, cap = layer.plan(S)
ids = ids.cpu().numpy()[:, 0]; sl = slots.cpu().numpy()[:, 0]
print("drop", (sl < 0).mean(), "load", load.cpu().numpy()[:20])
d = (outs[True].float() - outs[False].float()).abs()
print("fused vs unfused max", d.max().item())
lg = logits.double().cpu().numpy()
x64 = x.double().cpu().numpy()
for e in [0, 1, 5, 64, 127] + list(np.argsort(load.cpu().numpy())[-3:]):
    e = int(e)
    ex = [None] * E
    ex[e] = (w1[e].double().cpu().numpy(), b1[e].double().cpu().numpy(), w2[e].double().cpu().numpy(), b2[e].double().cpu().numpy())
    tok, want = O.forward_layer_sampled(x64, lg, ex, None, E, 1, 1.0, [e])
    kept = tok[sl[tok] >= 0]
    for fuse in (True, False):
        got = outs[fuse][torch.as_tensor(tok, device=dev)].double().cpu().numpy()
        err = np.abs(got - want)
        i = np.unravel_index(err.argmax(), err.shape)
        t = tok[i[0]]
        print(f"e={e} load={int(load[e])} fuse={fuse} maxerr={err.max():.4f} at tok {t} slot {sl[t]} col {i[1]} want {want[i]:.4f} got {got[i]:.4f} x {x64[t, i[1]]:.4f} p {np.exp(lg[t]-lg[t].max())[e]/np.exp(lg[t]-lg[t].max()).sum():.4f}")
