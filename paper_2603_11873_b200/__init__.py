"""AdaFuse hot path on B200: pre-gating router, fused switch, bs=1 decode.

The public surface mirrors /root/reference/pkg/src/lorafuse/__init__.py:75-133 for every
symbol on the hot path and adds the names BASELINE.json uses
(``pregate``, ``fused_switch``, ``merge``, ``unmerge``).  All compute runs in hand-written
sm_100a CUDA behind the C ABI of include/adafuse_b200.h; there is no CPU fallback.
"""

from .errors import (
    AliasingError,
    CalibrationError,
    ConfigError,
    DeviceError,
    DimensionError,
    InputError,
    PrecisionError,
    StateError,
)
from .linalg import (
    DEFAULT_TILE,
    EVENT_KINDS,
    DeviceTable,
    DispatchEvent,
    DispatchRecorder,
    DispatchSummary,
    Matrix,
    Segment,
    SegmentTable,
    TileConfig,
    gemm,
    gemm_accumulate_inplace,
    sgmm,
    sgmm_sequential,
)
from .routing import (
    DeviceDecision,
    GateDecision,
    RouterParams,
    pre_gate,
    pregate,
    pregate_device,
    route,
    router_logits,
)
from .adapters import (
    ConcatAdapter,
    ExpertBank,
    LoraExpert,
    SegmentGroup,
    SwitchTable,
    build_switch,
    concat_gated,
    expert_apply,
    load_bank,
    merge_all,
    save_bank,
)
from .model import (
    DecodeState,
    DecoderModel,
    ModelConfig,
    Strategy,
    build_model,
    decode_step,
    finalize_generation,
    forward_layer,
    fused_switch,
    generate,
    load_checkpoint,
    max_backbone_deviation,
    merge,
    prefill,
    save_checkpoint,
    unmerge,
    weights_digest,
)

__version__ = "0.1.0"
