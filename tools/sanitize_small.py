"""Small layer forwards for compute-sanitizer (one tool per call): k=1 fused
GEMM2 combine, k=2 standalone combine, Residual-MoE grouped launch (device
counter wait between expert and shared tiles), NaN rows, CUDA-graph replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05596_b200 import arch as A  # noqa: E402
from paper_2201_05596_b200.gating import GatingConfig  # noqa: E402

for (S, M, E, k, cf, res) in [(1000, 256, 8, 1, 1.0, False), (700, 128, 4, 2, 1.25, False),
                              (1500, 256, 4, 1, 1.0, True), (900, 128, 4, 2, 1.1, True)]:
    spec = A.LayerSpec(kind="moe", hidden=M, experts=E, residual=res, gating=GatingConfig(E, k, cf))
    p = A.init_layer_params(spec, np.random.default_rng(S))
    layer = A.MoeLayer(spec, p, dtype=torch.bfloat16)
    x = torch.randn(S, M, device="cuda").to(torch.bfloat16)
    x[3] = float("nan")
    y = layer(x)
    g = layer.graphed(S)
    y2 = g(x)
    torch.cuda.synchronize()
    print("ok", S, M, E, k, res, bool(torch.isfinite(y[:3]).all()))
