"""B200-native (sm_100a) DeepSpeed-MoE layer forward, drop-in for moekit's
gating / layer API (arXiv 2201.05596). See DESIGN.md and INTEGRATION.md."""

from . import arch, gating, tensor  # noqa: F401
from .arch import (  # noqa: F401
    FFN_MULT, FfnParams, LayerSpec, MoeLayer, MoeLayerParams, ValidationError, forward_ffn,
    forward_layer, init_layer_params, load_balance_loss,
)
from .gating import (  # noqa: F401
    DROPPED, DispatchPlan, ExpertBuffers, GatingConfig, OpCounter, TopKGate, build_dispatch_plan,
    combine_tokens, exclusive_scan_blelloch, scatter_tokens, top_k_gate,
)
from .tensor import ShapeError, Tensor  # noqa: F401

__version__ = "0.1.0"
