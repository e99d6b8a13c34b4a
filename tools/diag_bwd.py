"""Diagnostic: per-component backward error at one shape (GPU vs oracle)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2201_05596_b200 import arch as A
from paper_2201_05596_b200.gating import GatingConfig
from oracle import moe_oracle as O

S, M, E, k, cf, res = 3000, 512, 8, 1, 0.7, False
spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=res, gating=GatingConfig(E, k, cf))
rng = np.random.default_rng(S + E)
p = A.init_layer_params(spec, rng)
bf = lambda a: torch.as_tensor(a).to(torch.bfloat16).double().numpy()
for leaf in [p.gate_w] + [f.w1 for f in p.experts] + [f.w2 for f in p.experts]:
    leaf.value[:] = bf(leaf.value)
x64 = bf(rng.standard_normal((S, M)))
g64 = bf(rng.standard_normal((S, M)))
layer = A.MoeLayer(spec, p, dtype=torch.bfloat16)
layer.forward_train(torch.as_tensor(x64).to("cuda", torch.bfloat16))
logits = layer._train_ctx["logits"].double().cpu().numpy()
gr = layer.backward(torch.as_tensor(g64).to("cuda", torch.bfloat16))
experts = [(f.w1.value, f.b1.value, f.w2.value, f.b2.value) for f in p.experts]
want = O.forward_layer_backward(x64, logits, p.gate_w.value, experts, None, E, k, cf, g64)
got = gr["x"].float().cpu().numpy()
err = np.abs(got - want["x"])
rms = np.sqrt(np.mean(want["x"] ** 2))
i, j = np.unravel_index(np.argmax(err - 2e-2 * (np.abs(want["x"]) + rms)), err.shape)
print("rms", rms, "max err", err.max(), "at", i, j, "got", got[i, j], "want", want["x"][i, j])
ids, _, probs = O.top_k_gate(logits, E, k)
slots, _, _ = O.build_dispatch_plan_fast(ids, E, k, cf)
print("token", i, "ids", ids[i], "slots", slots[i], "probs", probs[i], "logits", logits[i])
# the gate term alone
dprobs = np.zeros_like(probs)
kept = slots != -1
for e in range(E):
    w1, b1, w2, b2 = experts[e]
    sel = np.nonzero(kept & (ids == e))[0]
    y = O.gelu(x64[sel] @ w1 + b1) @ w2 + b2
    dprobs[sel, e] = (g64[sel] * y).sum(1)
dl = probs * (dprobs - (dprobs * probs).sum(1, keepdims=True))
gate_term = dl @ p.gate_w.value.T
print("gate term rms", np.sqrt(np.mean(gate_term ** 2)), "at token", gate_term[i, j], "dl", dl[i])
print("per-row err rms top5:", np.sort(np.sqrt(np.mean(err ** 2, 1)))[-5:])
print("dgate", np.abs(gr["gate_w"].float().cpu().numpy() - want["gate_w"]).max(), np.abs(want["gate_w"]).max())
