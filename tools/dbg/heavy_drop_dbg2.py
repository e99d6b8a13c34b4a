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
layer = A.MoeLayer(spec, p, dtype=torch.bfloat16)
x = torch.randn(S, M, device=dev, generator=gen).to(torch.bfloat16)
x[:, 0] = 1.0
logits = torch.empty(S, E, device=dev)
out = layer(x, logits_out=logits)
torch.cuda.synchronize()
ws = layer._ws[S]
ids, gp, slots, load, cap = layer.plan(S)
sl = slots.cpu().numpy()[:, 0]
dropped = sl < 0
lg = logits.double().cpu().numpy()
x64 = x.double().cpu().numpy()
ld = load.cpu().numpy()
order = np.argsort(ld, kind="stable")
subset = sorted(set(int(e) for e in np.linspace(0, E - 1, 12).astype(int)) | {int(order[0]), int(order[-1]), int(order[E // 2]), int(order[-2])})
subset = subset[:16] if len(subset) >= 16 else subset + [e for e in range(E) if e not in subset][:16 - len(subset)]
print("subset", subset)
idsn = ids.cpu().numpy()[:, 0]
for e in subset:
    ex = [None] * E
    W1 = w1[e].double().cpu().numpy(); W2 = w2[e].double().cpu().numpy()
    B1 = b1[e].double().cpu().numpy(); B2 = b2[e].double().cpu().numpy()
    ex[e] = (W1, B1, W2, B2)
    tok, want = O.forward_layer_sampled(x64, lg, ex, None, E, 1, 1.0, [e])
    kt = ~dropped[tok]
    tk = tok[kt]; wk = want[kt]
    got = out[torch.as_tensor(tk, device=dev)].double().cpu().numpy()
    err = np.abs(got - wk)
    rms = 2.656
    exc = err - 0.02 * (np.abs(wk) + rms)
    i = np.unravel_index(exc.argmax(), exc.shape)
    t = tk[i[0]]; c = i[1]
    s = sl[t]
    hrow = ws["h"][e * cap + s].double().cpu().numpy()
    a = x64[t] @ W1 + B1[0]
    h_ref = O.gelu(a)
    y_from_gpu_h = hrow @ W2[:, c] + B2[0, c]
    y_ref = h_ref @ W2[:, c] + B2[0, c]
    pe = float(gp[t, 0])
    print(f"e={e} load={ld[e]} worst excess {exc.max():.4f} err {err[i]:.4f} tok {t} slot {s} col {c} want {wk[i]:.4f} got {got[i]:.4f} x {x64[t,c]:.3f} p {pe:.4f}"
          f" | y_ref {y_ref:.4f} y(gpu h) {y_from_gpu_h:.4f} h maxrelerr {np.max(np.abs(hrow-h_ref)/(np.abs(h_ref)+1e-3)):.4g} x+p*y(gpu h) {x64[t,c]+pe*y_from_gpu_h:.4f}")
