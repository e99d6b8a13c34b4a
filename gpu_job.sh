cat > /tmp/sanit.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2201_05596_b200 import arch as A, gating as G
from paper_2201_05596_b200.gating import GatingConfig
# routing API kernels (f64 + f32), plan, scan, scatter/combine
rng = np.random.default_rng(0)
cfg = GatingConfig(16, 2, 1.25)
lg = rng.standard_normal((1000, 16))
gate = G.top_k_gate(lg, cfg); plan = G.build_dispatch_plan(gate, cfg, 1000)
b = G.scatter_tokens(rng.standard_normal((1000, 24)), plan); G.combine_tokens(b, plan)
G.exclusive_scan_blelloch(rng.integers(0, 9, 70000)); G.exclusive_scan_blelloch(rng.standard_normal(100))
A.load_balance_loss(plan, gate.probs)
# layer forward: bf16 (tcgen05 gate + 2-CTA grouped GEMMs, fused combine), k=2 + residual, fp32
for k, res, dt in [(1, False, torch.bfloat16), (2, True, torch.bfloat16), (2, False, torch.float32)]:
    spec = A.LayerSpec(kind="moe", hidden=256, experts=8, residual=res, gating=GatingConfig(8, k, 1.0))
    p = A.init_layer_params(spec, np.random.default_rng(1))
    layer = A.MoeLayer(spec, p, dtype=dt, aux_loss=True)
    layer(torch.randn(700, 256, device="cuda").to(dt))
torch.cuda.synchronize(); print("sanitizer workload done")
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/sanit.py > gpurun_out/memcheck.log 2>&1; tail -15 gpurun_out/memcheck.log
