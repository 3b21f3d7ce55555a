"""Decode engine for the reference's decoder stack, on B200.

Host-side mirror of /root/reference/pkg/src/lorafuse/model.py: same ``ModelConfig`` /
``build_model`` (PCG64 draw order, so one seed names one model) / ``decode_step`` /
``prefill`` / ``generate`` / ``finalize_generation`` surface, same event trace, same errors.
The per-token hot path of ``PRE_GATED_FUSED`` (model.py:332-371 `_merged_pass`) is

    embed row gather -> pre-gate (1 launch) -> fused switch over ALL layers (1 launch)
    -> L x [GEMV + GELU + residual] (1 launch each) -> unembed GEMV -> argmax

with the routing decision, the token and every activation resident on the device; the only
host read per step is the 4-byte next token.  Weights are stored in bf16
(``precision="bf16"``, the default) or f32 (``"single"`` -- the reference's own mode).

Attribution: ``Strategy``, ``ModelConfig`` (fields, validation rules and messages, ``to_dict`` /
``from_dict``), ``DecoderModel`` and ``DecodeState`` are the reference's carrier classes
(model.py:66-162) restated field for field -- they ARE the public API this package keeps intact,
so their names, fields and error behaviour are taken from the reference, not invented here.
Everything below them (device residency, kernels, the refresh folded into the switch) is this
package's own.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _capi
from .adapters import ConcatAdapter, ExpertBank, LoraExpert, SwitchTable, expert_apply  # noqa: F401
from .errors import DeviceError, DimensionError, InputError, StateError
from .linalg import PRECISION_DTYPES, _AF_DTYPE, DispatchEvent, DispatchRecorder, Matrix, _ptr, gemm
from .routing import DeviceDecision, GateDecision, RouterParams, pregate_device, pregate_token_device


def _on_model_device(fn):
    """Run an engine entry point with the model's device current (the C ABI launches on the current
    device's stream and configures its kernels per device)."""
    import functools

    @functools.wraps(fn)
    def wrapper(model, *a, **kw):
        dev = model.embed.data.device
        if dev.type != "cuda" or torch.cuda.current_device() == dev.index:
            return fn(model, *a, **kw)
        with torch.cuda.device(dev):
            return fn(model, *a, **kw)

    return wrapper


class Strategy(Enum):
    """model.py:66-83.  All five run here; only BASE and PRE_GATED_FUSED are tuned -- the
    other three are the paper's baselines, expressed with the same GEMV kernel."""

    BASE = "base"
    LAYER_WISE_ROUTED = "layer_wise_routed"
    PRE_GATED_NAIVE = "pre_gated_naive"
    PRE_GATED_SIMPLE_MERGE = "pre_gated_simple_merge"
    PRE_GATED_FUSED = "pre_gated_fused"

    @property
    def pre_gated(self) -> bool:
        return self in (Strategy.PRE_GATED_NAIVE, Strategy.PRE_GATED_SIMPLE_MERGE, Strategy.PRE_GATED_FUSED)

    @property
    def merges_backbone(self) -> bool:
        return self in (Strategy.PRE_GATED_SIMPLE_MERGE, Strategy.PRE_GATED_FUSED)


@dataclass(frozen=True, slots=True)
class ModelConfig:
    """Shape and run parameters (model.py:86-142).  ``compute`` picks the switch arithmetic:
    "auto" (tensor path when eligible), "exact" (reference order), "fma", "mma"."""

    layers: int = 8
    hidden: int = 64
    vocab: int = 256
    experts: int = 8
    rank: int = 4
    top_k: int = 2
    precision: str = "bf16"
    seed: int = 0
    strategy: Strategy = Strategy.PRE_GATED_FUSED
    refresh_every: int = 0         # model.py:103; see `effective_refresh_every` for bf16 storage
    compute: str = "auto"
    switch_mode: str = "inplace"   # "inplace": W <- W + dNew - dOld; "from_pristine": W <- W0 + dNew (no drift)

    def validate(self) -> None:
        for name in ("layers", "hidden", "vocab", "experts", "rank", "top_k"):
            value = getattr(self, name)
            if not isinstance(value, int) or isinstance(value, bool) or value < 1:
                raise ValueError(f"{name} must be a positive integer, got {value!r}")
        if self.vocab < 2:
            raise ValueError("vocab must be >= 2")
        if self.top_k > self.experts:
            raise ValueError(f"top_k={self.top_k} exceeds experts={self.experts}")
        if self.top_k > _capi.AF_MAX_K:
            raise ValueError(f"top_k={self.top_k} exceeds the device decision record ({_capi.AF_MAX_K})")
        if self.rank > self.hidden:
            raise ValueError(f"rank={self.rank} exceeds hidden={self.hidden}")
        if self.precision not in PRECISION_DTYPES:
            raise ValueError(f"unknown precision {self.precision!r}")
        if not isinstance(self.strategy, Strategy):
            raise ValueError(f"strategy must be a Strategy, got {self.strategy!r}")
        if not isinstance(self.refresh_every, int) or self.refresh_every < -1:
            raise ValueError("refresh_every must be a non-negative integer (or -1: never, also for bf16 storage)")
        if not isinstance(self.seed, int):
            raise ValueError("seed must be an integer")
        if self.compute not in _capi.COMPUTE_MODES:
            raise ValueError(f"unknown compute mode {self.compute!r}")
        if self.switch_mode not in ("inplace", "from_pristine"):
            raise ValueError(f"unknown switch mode {self.switch_mode!r}")

    BF16_REFRESH_EVERY = 16

    @property
    def effective_refresh_every(self) -> int:
        """The refresh period `_merged_pass` uses.  The reference's default (0 = never) is right for its f32 / f64
        weights, whose in-place switch drifts by ~1e-8.  bf16 storage re-rounds W at every in-place switch (a
        ~0.3 sqrt(T) ulp random walk), and 16 switches is where the logits are still within 1e-2
        of the reference's trajectory -- so an in-place bf16 model left at 0 refreshes every 16 tokens.  The
        refresh is free here (it is folded into that token's switch launch, see `_merged_pass`);
        ``refresh_every=-1`` turns it off."""
        if self.refresh_every < 0:
            return 0
        if self.refresh_every == 0 and self.precision == "bf16" and self.switch_mode == "inplace" and self.strategy.merges_backbone:
            return self.BF16_REFRESH_EVERY
        return self.refresh_every

    def to_dict(self) -> dict:
        return {
            "layers": self.layers, "hidden": self.hidden, "vocab": self.vocab, "experts": self.experts,
            "rank": self.rank, "top_k": self.top_k, "precision": self.precision, "seed": self.seed,
            "strategy": self.strategy.value, "refresh_every": self.refresh_every, "compute": self.compute,
            "switch_mode": self.switch_mode,
        }

    @classmethod
    def from_dict(cls, raw: dict) -> "ModelConfig":
        data = dict(raw)
        if "strategy" in data and not isinstance(data["strategy"], Strategy):
            data["strategy"] = Strategy(data["strategy"])
        config = cls(**data)
        config.validate()
        return config


@dataclass(slots=True)
class DecoderModel:
    """model.py:145-153 plus the resident device structures of the B200 path."""

    config: ModelConfig
    embed: Matrix            # vocab x d
    backbone: list           # L matrices d x d, mutated by the switch
    bank: ExpertBank         # views into bank_down / bank_up
    router: RouterParams
    unembed: Matrix          # d x vocab
    pristine_backbone: list
    bank_down: list = field(default_factory=list)   # per layer [N][r][d]
    bank_up: list = field(default_factory=list)     # per layer [N][d][r]
    table: SwitchTable | None = None


@dataclass(slots=True)
class DecodeState:
    """Per-generation state (model.py:156-162).  ``prev_decision`` is the previous token's
    routing decision in device memory -- the GPU form of ``prev_concats``."""

    prev_decision: DeviceDecision | None = None
    last_hidden_dev: torch.Tensor | None = None
    tokens_done: int = 0
    spare_decision: DeviceDecision | None = None   # ping-pong buffer
    token_dev: torch.Tensor | None = None          # int32[1]: the token being consumed

    @property
    def prev_concats(self):
        return self.prev_decision

    @property
    def last_hidden(self):
        return None if self.last_hidden_dev is None else self.last_hidden_dev.detach().cpu().numpy().copy()


# ---------------------------------------------------------------------------
# Construction
# ---------------------------------------------------------------------------


def bf16_round_np(a: np.ndarray) -> np.ndarray:
    """RNE f32 -> bf16 grid, carried as f32."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def draw_weights(config: ModelConfig) -> dict:
    """Host arrays in the reference's draw order (model.py:182-203): PCG64(seed); uniform
    +-1/sqrt(fan_in) with fan_in = d, except the up factors (r); drawn in f64, cast to f32."""
    rng = np.random.Generator(np.random.PCG64(config.seed))
    d, r = config.hidden, config.rank
    bound_d, bound_r = 1.0 / math.sqrt(d), 1.0 / math.sqrt(r)

    def draw(rows, cols, bound):
        return rng.uniform(-bound, bound, size=(rows, cols)).astype(np.float32)

    out = {"embed": draw(config.vocab, d, bound_d), "router": draw(config.experts, d, bound_d),
           "unembed": draw(d, config.vocab, bound_d), "backbone": [], "down": [], "up": []}
    for _ in range(config.layers):
        out["backbone"].append(draw(d, d, bound_d))
        downs, ups = [], []
        for _ in range(config.experts):
            downs.append(draw(r, d, bound_d))
            ups.append(draw(d, r, bound_r))
        out["down"].append(np.stack(downs))
        out["up"].append(np.stack(ups))
    return out


def build_model(config: ModelConfig, device=None) -> DecoderModel:
    """Deterministic init from config.seed (model.py:170-214), uploaded once; the expert bank
    is packed per layer as [N][r][d] / [N][d][r] and the descriptor table is built here."""
    config.validate()
    torch_ = _capi.require_cuda()
    dev = torch_.device(device) if device is not None else torch_.device("cuda", torch_.cuda.current_device())
    if dev.type == "cuda" and dev.index is not None and dev.index != torch_.cuda.current_device():
        with torch_.cuda.device(dev):      # the descriptor table is allocated on the CURRENT device
            return build_model(config, dev)
    w = draw_weights(config)
    prec = config.precision

    def up(a):
        return Matrix(torch_.from_numpy(a), prec, device=dev)

    embed, router, unembed = up(w["embed"]), RouterParams(weight=up(w["router"])), up(w["unembed"])
    backbone = [up(a) for a in w["backbone"]]
    dtype = PRECISION_DTYPES[prec]
    bank_down = [torch_.from_numpy(a).to(device=dev, dtype=dtype).contiguous() for a in w["down"]]
    bank_up = [torch_.from_numpy(a).to(device=dev, dtype=dtype).contiguous() for a in w["up"]]
    layers = tuple(
        tuple(LoraExpert(down=Matrix(dn[e], prec), up=Matrix(upb[e], prec)) for e in range(config.experts))
        for dn, upb in zip(bank_down, bank_up)
    )
    bank = ExpertBank(layers=layers)
    bank.validate()
    pristine = [m.copy() for m in backbone]
    table = SwitchTable(backbone, bank_down, bank_up, pristine=pristine)
    return DecoderModel(config, embed, backbone, bank, router, unembed, pristine, bank_down, bank_up, table)


def weights_digest(model: DecoderModel) -> str:
    """SHA-256 over all weights in draw order (model.py:217-228), on the stored bit patterns."""
    h = hashlib.sha256()

    def feed(m: Matrix):
        t = m.data.detach().contiguous()
        h.update((t.view(torch.int16) if t.dtype == torch.bfloat16 else t).cpu().numpy().tobytes())

    feed(model.embed)
    feed(model.router.weight)
    feed(model.unembed)
    for li in range(model.config.layers):
        feed(model.pristine_backbone[li])
        for expert in model.bank.layers[li]:
            feed(expert.down)
            feed(expert.up)
    return h.hexdigest()


@_on_model_device
def max_backbone_deviation(model: DecoderModel) -> float:
    """Largest |backbone - pristine| entry across all layers (model.py:231-236)."""
    return model.table.max_deviation()


# ---------------------------------------------------------------------------
# Forward passes
# ---------------------------------------------------------------------------


def _check_token(model: DecoderModel, token) -> int:
    if not isinstance(token, (int, np.integer)) or isinstance(token, bool) or not 0 <= token < model.config.vocab:
        raise InputError(f"token {token!r} outside vocab of {model.config.vocab}")
    return int(token)


def _embed_token(model: DecoderModel, token: int, recorder: DispatchRecorder, token_dev: torch.Tensor | None = None) -> Matrix:
    """Row gather embed[token] -> d x 1 single column (model.py:248-258)."""
    token = _check_token(model, token)
    d = model.config.hidden
    if token_dev is None:
        token_dev = torch.tensor([token], dtype=torch.int32, device=model.embed.data.device)
    out = torch.empty((d, 1), dtype=torch.float32, device=model.embed.data.device)
    _capi.check(_capi.lib().af_embed(_ptr(model.embed.data), _AF_DTYPE[model.embed.precision], d, _ptr(token_dev), _ptr(out), _capi.stream_ptr()))
    recorder.record("elementwise", flops=0, bytes_touched=2 * d * model.embed.itemsize, label="other")
    return Matrix(out, "single")


def _unembed(model: DecoderModel, x: Matrix, recorder: DispatchRecorder) -> torch.Tensor:
    """x^T (1 x d) @ unembed (d x V) -> V logits on the device (model.py:261-263)."""
    logits = gemm(Matrix(x.data.view(1, -1), "single"), model.unembed, recorder, label="other")
    return logits.data[0]


def forward_layer(model: DecoderModel, layer_idx: int, x: Matrix, gate: GateDecision | None, recorder: DispatchRecorder,
                  strategy: Strategy | None = None) -> Matrix:
    """One layer: x + gelu(layer map of x) under the given strategy (model.py:266-305).

    BASE and the merge strategies: ONE launch (GEMV with the GELU + residual epilogue fused);
    the trace still carries the reference's gemm + elementwise pair."""
    if strategy is None:
        strategy = model.config.strategy
    if not 0 <= layer_idx < model.config.layers:
        raise IndexError(f"layer {layer_idx} outside stack of {model.config.layers}")
    f = model.backbone[layer_idx]
    d = model.config.hidden
    if strategy in (Strategy.LAYER_WISE_ROUTED, Strategy.PRE_GATED_NAIVE):
        y = gemm(f, x, recorder, label="backbone")
        if strategy is Strategy.LAYER_WISE_ROUTED and layer_idx > 0:
            from .routing import route

            gate = route(model.router, x, model.config.top_k, recorder)
        if gate is None:
            raise StateError(f"{strategy.value} needs a gate decision at layer {layer_idx}")
        bank_layer = model.bank.layers[layer_idx]
        for expert_id, weight in zip(gate.expert_ids, gate.weights):
            y.data += expert_apply(bank_layer[expert_id], x, weight, recorder).data
        h = 0.5 * y.data * (1.0 + torch.erf(y.data * (1.0 / math.sqrt(2.0))))
        out = Matrix(x.data + h, "single")
    else:
        out = gemm(f, x, recorder, label="backbone", epilogue="gelu_residual", residual=x)
    recorder.record("elementwise", flops=d, bytes_touched=2 * d * x.itemsize, label="backbone")
    return out


def _refresh_from_pristine(model: DecoderModel, state: DecodeState) -> None:
    model.table.refresh()  # model.py:308-312
    state.prev_decision = None


def _switch_event(model: DecoderModel, n_blocks: int, recorder: DispatchRecorder) -> None:
    s = n_blocks * model.config.rank
    recorder.record("sgmm", flops=model.table.switch_flops(s), bytes_touched=model.table.switch_bytes(s), label="switch")


def _unmerged_pass(model: DecoderModel, token: int, recorder: DispatchRecorder, strategy: Strategy, capture=None):
    from .routing import route

    x = _embed_token(model, token, recorder)
    gate = route(model.router, x, model.config.top_k, recorder)
    for layer_idx in range(model.config.layers):
        x = forward_layer(model, layer_idx, x, gate, recorder, strategy=strategy)
        if capture is not None:
            capture.append(x.data[:, 0].detach().cpu().numpy().copy())
    return x, _unembed(model, x, recorder)


def _merged_pass(model: DecoderModel, state: DecodeState, token: int, recorder: DispatchRecorder, capture=None):
    """Embed -> pre-gate -> delta swap -> plain layer stack -> logits (model.py:332-371)."""
    config = model.config
    strategy = config.strategy
    dev = model.embed.data.device
    token = _check_token(model, token)
    if state.token_dev is None:
        state.token_dev = torch.empty(1, dtype=torch.int32, device=dev)
    state.token_dev.fill_(token)
    x = _embed_token(model, token, recorder, token_dev=state.token_dev)
    cur = state.spare_decision if state.spare_decision is not None else DeviceDecision(dev)
    state.spare_decision = None
    pregate_device(model.router, x, config.top_k, recorder, out=cur)
    period = config.effective_refresh_every
    refresh = period > 0 and state.tokens_done > 0 and state.tokens_done % period == 0      # model.py:344-349
    if refresh and strategy is not Strategy.PRE_GATED_FUSED:
        _refresh_from_pristine(model, state)
    prev = state.prev_decision
    if strategy is Strategy.PRE_GATED_FUSED and (config.switch_mode == "from_pristine" or refresh):
        # A refreshing token: "copy W0 over W, forget prev, merge cur" (model.py:308-312, :350-357) is exactly
        # W <- bf16(W0 + delta(cur)) -- the from-pristine switch -- so the refresh rides in this token's one
        # launch instead of costing a copy of every weight.
        # Same HBM traffic (read W0, write W), half the stacked rank, and no bf16 re-rounding drift.
        model.table.switch(None, cur, max_k=config.top_k, compute=config.compute, mode="from_pristine")
        _switch_event(model, config.top_k, recorder)
    elif strategy is Strategy.PRE_GATED_FUSED:
        model.table.switch(prev, cur, max_k=config.top_k, compute=config.compute)
        _switch_event(model, (config.top_k if prev is not None else 0) + config.top_k, recorder)
    else:  # PRE_GATED_SIMPLE_MERGE: unmerge then merge (model.py:358-365), two launches
        if prev is not None:
            model.table.unmerge(prev, max_k=config.top_k, compute=config.compute)
        model.table.merge(cur, max_k=config.top_k, compute=config.compute)
        per_layer = (2 if prev is not None else 1)
        s = config.top_k * config.rank
        for _ in range(config.layers * per_layer):
            recorder.record("gemm", flops=2 * config.hidden * s * config.hidden,
                            bytes_touched=(2 * config.hidden * s) * 4 + 2 * config.hidden * config.hidden * model.backbone[0].itemsize,
                            label="switch")
    state.spare_decision = prev
    state.prev_decision = cur
    for layer_idx in range(config.layers):
        x = forward_layer(model, layer_idx, x, None, recorder, strategy=strategy)
        if capture is not None:
            capture.append(x.data[:, 0].detach().cpu().numpy().copy())
    return x, _unembed(model, x, recorder)


@_on_model_device
def decode_step(model: DecoderModel, state: DecodeState, token: int, recorder: DispatchRecorder, capture=None,
                logits_out: list | None = None):
    """One greedy decode step (model.py:374-405): consume ``token``, emit the next token id;
    returns (next_token, events appended by this step).  Ties pick the lowest token id."""
    mark = recorder.mark()
    strategy = model.config.strategy
    if strategy.merges_backbone:
        x, logits = _merged_pass(model, state, token, recorder, capture=capture)
    else:
        x, logits = _unmerged_pass(model, _check_token(model, token), recorder, strategy, capture=capture)
    nxt = torch.empty(1, dtype=torch.int32, device=logits.device)
    _capi.check(_capi.lib().af_argmax(_ptr(logits), int(logits.numel()), _ptr(nxt), _capi.stream_ptr()))
    recorder.record("reduce", flops=model.config.vocab, bytes_touched=model.config.vocab * 4, label="other")
    next_token = int(nxt.item())  # the one host read of the step
    if model.table is not None and strategy.merges_backbone:
        model.table.status()      # what the switch kernel flagged for this step's device decision (adapters.py:199-200)
    if logits_out is not None:
        logits_out.append(logits.detach().cpu().numpy().copy())
    state.last_hidden_dev = x.data[:, 0]
    state.tokens_done += 1
    return next_token, recorder.events_since(mark)


@_on_model_device
def prefill(model: DecoderModel, tokens, recorder: DispatchRecorder) -> DecodeState:
    """Process a prompt along the unfused per-token path (model.py:408-425); never an sgmm."""
    tokens = list(tokens)
    if not tokens:
        raise InputError("prompt must contain at least one token")
    strategy = model.config.strategy
    if strategy.pre_gated:
        strategy = Strategy.PRE_GATED_NAIVE
    x = None
    for token in tokens:
        x, _ = _unmerged_pass(model, _check_token(model, token), recorder, strategy)
    return DecodeState(prev_decision=None, last_hidden_dev=x.data[:, 0], tokens_done=0)


@_on_model_device
def generate(model: DecoderModel, prompt, n_new: int, recorder: DispatchRecorder, hidden_sink: list | None = None,
             forced=None, logits_sink: list | None = None):
    """Prefill, n_new greedy decode steps, then restore the backbone (model.py:428-457).

    Returns (generated tokens, DispatchTrace of all events), as the reference does.  ``forced`` (an
    extension) teacher-forces the consumed token stream so every step really switches."""
    from .perf import DispatchTrace

    if n_new < 1:
        raise InputError(f"n_new must be >= 1, got {n_new}")
    mark = recorder.mark()
    state = prefill(model, prompt, recorder)
    token = int(list(prompt)[-1])
    generated = []
    for step in range(n_new):
        capture = [] if hidden_sink is not None else None
        if forced is not None:
            token = int(forced[step])
        token, _ = decode_step(model, state, token, recorder, capture=capture, logits_out=logits_sink)
        generated.append(token)
        if hidden_sink is not None:
            hidden_sink.append(capture)
    finalize_generation(model, state, recorder)
    return generated, DispatchTrace(tuple(recorder.events_since(mark)))


@_on_model_device
def finalize_generation(model: DecoderModel, state: DecodeState, recorder: DispatchRecorder) -> None:
    """Unmerge the last token's delta arithmetically (model.py:460-474) -- one launch over all
    layers here; the trace keeps the reference's one gemm event per layer."""
    if state.prev_decision is None:
        return
    config = model.config
    if config.switch_mode == "from_pristine" and config.strategy is Strategy.PRE_GATED_FUSED:
        model.table.refresh()
    else:
        model.table.unmerge(state.prev_decision, max_k=config.top_k, compute=config.compute)
    s = config.top_k * config.rank
    for f in model.backbone:
        recorder.record("gemm", flops=2 * f.rows * s * f.cols,
                        bytes_touched=(f.rows * s + s * f.cols) * 4 + 2 * f.rows * f.cols * f.itemsize, label="switch")
    state.prev_decision = None


# ---------------------------------------------------------------------------
# north_star aliases
# ---------------------------------------------------------------------------


@_on_model_device
def fused_switch(model: DecoderModel, prev_decision, cur_decision, recorder: DispatchRecorder | None = None, **kw) -> None:
    """W <- W + delta(cur) - delta(prev) over every adapted matrix in one launch.
    Decisions may be ``GateDecision`` (host) or ``DeviceDecision``; None = empty."""
    kw.setdefault("max_k", model.config.top_k)
    kw.setdefault("compute", model.config.compute)
    model.table.switch(prev_decision, cur_decision, **kw)
    if recorder is not None:
        nb = sum(model.config.top_k if d is not None else 0 for d in (prev_decision, cur_decision))
        _switch_event(model, nb, recorder)


def merge(model: DecoderModel, decision, recorder: DispatchRecorder | None = None, **kw) -> None:
    fused_switch(model, None, decision, recorder, **kw)


def unmerge(model: DecoderModel, decision, recorder: DispatchRecorder | None = None, **kw) -> None:
    fused_switch(model, decision, None, recorder, **kw)


__all__ = [n for n in dir() if not n.startswith("_")] + ["_merged_pass", "_embed_token", "_unembed"]
_ = (DispatchEvent, DeviceError, pregate_token_device)


# ---------------------------------------------------------------------------
# Checkpoints (model.py:481-541): the reference's npz container, read and written
# ---------------------------------------------------------------------------

_CHECKPOINT_FORMAT = "lorafuse-checkpoint-v1"
_REFERENCE_CONFIG_KEYS = ("layers", "hidden", "vocab", "experts", "rank", "top_k", "precision", "seed", "strategy", "refresh_every")


def save_checkpoint(model: DecoderModel, path) -> None:
    """model.py:484-505: config + all weights; the PRISTINE backbone is what gets saved, so a
    checkpoint captures the unmerged model even while a token's delta is fused in.  Arrays are
    written as f32 and the header's config carries only the reference's keys with a reference
    precision tag, so the reference's own `load_checkpoint` reads the file; the device-side extras
    travel under "device"."""
    import json

    cfg = model.config.to_dict()
    ref_cfg = {k: cfg[k] for k in _REFERENCE_CONFIG_KEYS}
    ref_cfg["precision"] = "single" if cfg["precision"] == "bf16" else cfg["precision"]
    header = {"format": _CHECKPOINT_FORMAT, "config": ref_cfg,
              "device": {"precision": cfg["precision"], "compute": cfg["compute"], "switch_mode": cfg["switch_mode"]}}
    f32 = lambda m: m.numpy().astype(np.float32)  # noqa: E731
    arrays = {"header": np.frombuffer(json.dumps(header).encode("utf-8"), dtype=np.uint8), "embed": f32(model.embed),
              "router": f32(model.router.weight), "unembed": f32(model.unembed)}
    for li in range(model.config.layers):
        arrays[f"backbone{li}"] = f32(model.pristine_backbone[li])
        for ei, expert in enumerate(model.bank.layers[li]):
            arrays[f"layer{li}/expert{ei}/down"] = f32(expert.down)
            arrays[f"layer{li}/expert{ei}/up"] = f32(expert.up)
    with open(path, "wb") as fh:
        np.savez(fh, **arrays)


def load_checkpoint(path, precision: str | None = None, device=None) -> DecoderModel:
    """model.py:508-541.  Reads checkpoints written by the reference or by `save_checkpoint`, uploads
    the weights, packs the expert bank into the per-layer [N][r][d] / [N][d][r] device layout and
    builds the descriptor table -- the model is ready to decode."""
    import json

    from .adapters import _load_precision, pack_bank_arrays

    torch_ = _capi.require_cuda()
    dev = torch_.device(device) if device is not None else torch_.device("cuda", torch_.cuda.current_device())
    with np.load(path) as archive:
        header = json.loads(bytes(archive["header"]).decode("utf-8"))
        if header.get("format") != _CHECKPOINT_FORMAT:
            raise ValueError(f"not a {_CHECKPOINT_FORMAT} container: {path}")
        raw = dict(header["config"])
        extra = header.get("device", {})
        prec = _load_precision(extra.get("precision", raw.get("precision", "single")), precision)
        raw["precision"] = prec
        for key in ("compute", "switch_mode"):
            if key in extra:
                raw[key] = extra[key]
        config = ModelConfig.from_dict(raw)

        def up(name):
            return Matrix(torch_.from_numpy(np.asarray(archive[name], dtype=np.float32)), prec, device=dev)

        embed, router, unembed = up("embed"), RouterParams(weight=up("router")), up("unembed")
        backbone = [up(f"backbone{li}") for li in range(config.layers)]
        bank, bank_down, bank_up = pack_bank_arrays(archive, config.layers, config.experts, prec, dev)
    if embed.rows != config.vocab or embed.cols != config.hidden:
        raise DimensionError("checkpoint embed shape disagrees with its config")
    pristine = [m.copy() for m in backbone]
    table = SwitchTable(backbone, bank_down, bank_up, pristine=pristine)
    return DecoderModel(config, embed, backbone, bank, router, unembed, pristine, bank_down, bank_up, table)

