"""Diagnose one training-path parity case: per-row dx error against the oracle,
with the rows' routing (expert, slot, kept) for the worst rows, repeated runs
(nondeterminism check). python tools/dbg/bwd_case_dbg.py S M E k cf res"""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import moe_oracle as O  # noqa: E402
from paper_2201_05596_b200 import arch as A  # noqa: E402
from paper_2201_05596_b200.gating import GatingConfig  # noqa: E402

S, M, E, k = (int(v) for v in sys.argv[1:5])
cf, res = float(sys.argv[5]), sys.argv[6] == "True"
spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=res, gating=GatingConfig(E, k, cf))
rng = np.random.default_rng(S + E)
p = A.init_layer_params(spec, rng)
bf = lambda a: torch.as_tensor(a).to(torch.bfloat16).double().numpy()  # noqa: E731
for leaf in [p.gate_w] + [f.w1 for f in p.experts] + [f.w2 for f in p.experts] + (
        [p.shared.w1, p.shared.w2] if res else []):
    leaf.value[:] = bf(leaf.value)
x64 = bf(rng.standard_normal((S, M)))
g64 = bf(rng.standard_normal((S, M)))
layer = A.MoeLayer(spec, p, dtype=torch.bfloat16)
outs = []
for rep in range(3):
    layer.forward_train(torch.as_tensor(x64).to("cuda", torch.bfloat16))
    logits = layer._train_ctx["logits"].double().cpu().numpy()
    gr = layer.backward(torch.as_tensor(g64).to("cuda", torch.bfloat16))
    outs.append(gr["x"].float().cpu().numpy())
print("dx deterministic across runs:", all(np.array_equal(outs[0], o) for o in outs[1:]))
c = layer._train_ctx
ids = c["ids"].cpu().numpy()
slots = c["slots"].cpu().numpy()
experts = [(f.w1.value, f.b1.value, f.w2.value, f.b2.value) for f in p.experts]
shared = (p.shared.w1.value, p.shared.b1.value, p.shared.w2.value, p.shared.b2.value) if res else None
want = O.forward_layer_backward(x64, logits, p.gate_w.value, experts, shared, E, k, cf, g64)["x"]
got = outs[0].astype(np.float64)
rms = float(np.sqrt(np.mean(want ** 2)))
ex = np.abs(got - want) - 2e-2 * (np.abs(want) + rms)
row_ex = ex.max(axis=1)
order = np.argsort(-row_ex)[:12]
cap = c["cap"]
print("cap", cap, "rms", rms, "max excess", ex.max(), "rows over:", int((row_ex > 0).sum()))
rel = np.abs(got - want) / (np.abs(want) + rms)
print("relative error: median %.2e p99 %.2e max %.2e" % (np.median(rel), np.quantile(rel, 0.99), rel.max()))
for t in order:
    j = int(np.argmax(ex[t]))
    print(f"row {t} ids {ids[t]} slots {slots[t]} excess {row_ex[t]:.3e} col {j} got {got[t, j]:.4f} "
          f"want {want[t, j]:.4f} row rel err max {rel[t].max():.2e}")
