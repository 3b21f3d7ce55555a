"""Token-level pre-gating router.

Host-side mirror of /root/reference/pkg/src/lorafuse/routing.py.  One launch
(`af_pregate`, csrc/af_decode.cuh) does the router GEMV, the stable top-k and the softmax
over the selected logits; the decision is left in device memory as an `af_decision` so the
fused switch consumes it without a host round trip.  ``route``/``pre_gate`` keep the
reference's return type (an immutable ``GateDecision`` of Python ints/floats) and therefore
synchronise; ``pregate_device`` is the asynchronous form the decode loop uses.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from .errors import DeviceError, DimensionError
from .linalg import _AF_DTYPE, DispatchRecorder, Matrix, _ptr


@dataclass(frozen=True, slots=True)
class RouterParams:
    """Routing weights, one row of ``weight`` (N x d) per expert (routing.py:22-34)."""

    weight: Matrix

    @property
    def n_experts(self) -> int:
        return self.weight.rows

    @property
    def hidden(self) -> int:
        return self.weight.cols


@dataclass(frozen=True, slots=True)
class GateDecision:
    """Chosen experts and mixture weights (routing.py:37-46): ids by descending logit, ties by
    ascending index; weights strictly positive, summing to 1 (f32 arithmetic)."""

    expert_ids: tuple
    weights: tuple


DECISION_BYTES = ctypes.sizeof(_capi.Decision)


def decision_to_struct(gate: GateDecision | None) -> _capi.Decision | None:
    if gate is None:
        return None
    k = len(gate.expert_ids)
    if k > _capi.AF_MAX_K:
        raise ValueError(f"a decision holds at most {_capi.AF_MAX_K} experts, got {k}")
    d = _capi.Decision()
    d.k = k
    for j in range(k):
        d.ids[j] = int(gate.expert_ids[j])
        d.weights[j] = float(gate.weights[j])
    return d


class DeviceDecision:
    """An `af_decision` in device memory (128 bytes) -- the GPU form of ``GateDecision``."""

    __slots__ = ("buf",)

    def __init__(self, device=None, buf: torch.Tensor | None = None):
        if buf is None:
            if device is None:
                device = torch.device("cuda", torch.cuda.current_device())
            buf = torch.zeros(DECISION_BYTES, dtype=torch.uint8, device=device)
        self.buf = buf

    @property
    def ptr(self) -> int:
        return int(self.buf.data_ptr())

    @classmethod
    def from_host(cls, gate: GateDecision, device=None) -> "DeviceDecision":
        raw = bytes(decision_to_struct(gate))
        host = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
        out = cls(device)
        out.buf.copy_(host)
        return out

    def to_host(self) -> GateDecision:
        """Synchronising read-back."""
        raw = self.buf.cpu().numpy().tobytes()
        d = _capi.Decision.from_buffer_copy(raw)
        k = int(d.k)
        return GateDecision(tuple(int(d.ids[j]) for j in range(k)), tuple(float(d.weights[j]) for j in range(k)))


def _validate(router: RouterParams, x: Matrix, k: int) -> None:
    # routing.py:57-62: k first, then the shape of x
    if not 1 <= k <= router.n_experts:
        raise ValueError(f"k={k} must be in [1, {router.n_experts}]")
    if x.rows != router.hidden or x.cols != 1:
        raise DimensionError(f"router expects a {router.hidden}x1 hidden state, got {x.rows}x{x.cols}")


def _record(router: RouterParams, x: Matrix, recorder: DispatchRecorder) -> None:
    # one gemm + one elementwise event, both labelled "router" (routing.py:63, 69-74)
    n, d = router.n_experts, router.hidden
    recorder.record("gemm", flops=2 * n * d, bytes_touched=n * d * router.weight.itemsize + d * x.itemsize + n * 4, label="router")
    recorder.record("elementwise", flops=n, bytes_touched=2 * n * 4, label="router")


def pregate_device(router: RouterParams, x: Matrix, k: int, recorder: DispatchRecorder, out: DeviceDecision | None = None,
                   logits_out: torch.Tensor | None = None) -> DeviceDecision:
    """Asynchronous pre-gate: the decision stays on the device."""
    _validate(router, x, k)
    if not (router.weight.data.is_cuda and x.data.is_cuda):
        raise DeviceError("operand is not on a CUDA device: the B200 path has no CPU fallback")
    if out is None:
        out = DeviceDecision(x.data.device)
    _capi.check(
        _capi.lib().af_pregate(
            _ptr(router.weight.data), _AF_DTYPE[router.weight.precision], router.n_experts, router.hidden,
            _ptr(x.data), _AF_DTYPE[x.precision], None, k, out.ptr,
            _ptr(logits_out) if logits_out is not None else None, _capi.stream_ptr(),
        )
    )
    _record(router, x, recorder)
    return out


def pregate_token_device(router: RouterParams, embed: Matrix, token_dev: torch.Tensor, k: int, recorder: DispatchRecorder,
                         out: DeviceDecision) -> DeviceDecision:
    """Pre-gate fused with the embedding-row gather (model.py:342-343): routes on
    ``embed[*token_dev]`` without materialising the column."""
    if not 1 <= k <= router.n_experts:
        raise ValueError(f"k={k} must be in [1, {router.n_experts}]")
    if embed.cols != router.hidden:
        raise DimensionError(f"router expects a {router.hidden}x1 hidden state, got {embed.cols}x1")
    _capi.check(
        _capi.lib().af_pregate(
            _ptr(router.weight.data), _AF_DTYPE[router.weight.precision], router.n_experts, router.hidden,
            _ptr(embed.data), _AF_DTYPE[embed.precision], _ptr(token_dev), k, out.ptr, None, _capi.stream_ptr(),
        )
    )
    n, d = router.n_experts, router.hidden
    recorder.record("gemm", flops=2 * n * d, bytes_touched=n * d * router.weight.itemsize + d * embed.itemsize + n * 4, label="router")
    recorder.record("elementwise", flops=n, bytes_touched=2 * n * 4, label="router")
    return out


def route(router: RouterParams, x: Matrix, k: int, recorder: DispatchRecorder) -> GateDecision:
    """Score experts for one hidden state and pick the top k (routing.py:49-78)."""
    return pregate_device(router, x, k, recorder).to_host()


def pre_gate(router: RouterParams, x_first: Matrix, k: int, recorder: DispatchRecorder) -> GateDecision:
    """Route once on the hidden state entering the first expanded layer (routing.py:81-89)."""
    return route(router, x_first, k, recorder)


pregate = pre_gate  # the name BASELINE.json.north_star uses


def router_logits(router: RouterParams, x: Matrix) -> np.ndarray:
    """The N router logits of one hidden state (diagnostics: top-k margins)."""
    _validate(router, x, 1)
    logits = torch.empty(router.n_experts, dtype=torch.float32, device=x.data.device)
    pregate_device(router, x, 1, DispatchRecorder(), logits_out=logits)
    return logits.cpu().numpy()
