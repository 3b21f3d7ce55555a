"""Adapter algebra and the fused switch.

Host-side mirror of /root/reference/pkg/src/lorafuse/adapters.py.  Two forms live here:

* the reference's *materialised* algebra -- ``concat_gated`` / ``build_switch`` / ``merge_all``
  on ``ConcatAdapter`` objects -- kept with the same names, argument order, provenance and
  error behaviour so reference-style code and tests run unchanged (one sgmm launch per
  ``merge_all``);
* the B200 form the decode loop uses: ``SwitchTable`` -- the device-side descriptor table
  built ONCE at model load over the resident expert bank -- and ``fused_switch`` /
  ``merge`` / ``unmerge``, where a per-token decision (expert ids + gate weights, in device
  memory) selects bank blocks inside the kernel.  Nothing is concatenated, negated or copied
  per token: the gate is folded into the DOWN rows while they are staged in shared memory
  (adapters.py:202), previous blocks are negated there (adapters.py:230).

Attribution: ``LoraExpert``, ``ExpertBank`` and ``ConcatAdapter`` (fields, ``validate`` rules and their
messages, ``ConcatAdapter.empty``) and the bodies of ``concat_gated`` / ``build_switch`` are the
reference's (adapters.py:49-233) restated on torch tensors -- they are the public API this package
keeps intact and exist here for parity tests and reference-style callers.  ``SwitchTable``,
``SegmentGroup`` and the packed bank layout are this package's own and are what the decode loop runs.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _capi
from .errors import DeviceError, DimensionError, PrecisionError
from .linalg import (
    PRECISION_DTYPES,
    default_device,
    DEFAULT_TILE,
    DeviceTable,
    DispatchRecorder,
    Matrix,
    Segment,
    SegmentTable,
    TileConfig,
    _ptr,
    gemm,
    sgmm,
)
from .routing import DeviceDecision, GateDecision, decision_to_struct

# ---------------------------------------------------------------------------
# Expert containers (adapters.py:49-109)
# ---------------------------------------------------------------------------


@dataclass(frozen=True, slots=True)
class LoraExpert:
    """One rank-r factor pair for one backbone matrix: down = A (r x d_in), up = B (d_out x r)."""

    down: Matrix
    up: Matrix

    @property
    def rank(self) -> int:
        return self.down.rows

    def validate(self) -> None:
        if self.down.rows != self.up.cols:
            raise DimensionError(
                f"expert rank mismatch: down has {self.down.rows} rows, up has {self.up.cols} columns"
            )
        if self.down.rows < 1:
            raise DimensionError("expert rank must be >= 1")
        if self.down.precision != self.up.precision:
            raise PrecisionError("expert factors carry mixed precision tags")


@dataclass(frozen=True, slots=True)
class ExpertBank:
    """layers[l][i] adapts backbone matrix l; same expert count, rank and shape everywhere."""

    layers: tuple

    @property
    def n_layers(self) -> int:
        return len(self.layers)

    @property
    def n_experts(self) -> int:
        return len(self.layers[0])

    @property
    def rank(self) -> int:
        return self.layers[0][0].rank

    def validate(self) -> None:
        if not self.layers or not self.layers[0]:
            raise DimensionError("expert bank has no layers or no experts")
        n = len(self.layers[0])
        first = self.layers[0][0]
        for li, layer in enumerate(self.layers):
            if len(layer) != n:
                raise DimensionError(f"layer {li} holds {len(layer)} experts, expected {n}")
            for expert in layer:
                expert.validate()
                if expert.rank != first.rank:
                    raise DimensionError("experts must share one rank")
                if expert.down.cols != first.down.cols or expert.up.rows != first.up.rows:
                    raise DimensionError("experts must share one input/output shape")


# ---------------------------------------------------------------------------
# Concatenated adapters (adapters.py:117-162)
# ---------------------------------------------------------------------------


@dataclass(frozen=True, slots=True)
class ConcatAdapter:
    """Stacked expert blocks for one matrix: down_cat (s x d_in), up_cat (d_out x s);
    provenance = one (expert_id, gate_weight, sign) per block, gates live in DOWN only."""

    down_cat: Matrix
    up_cat: Matrix
    provenance: tuple

    @property
    def s(self) -> int:
        return self.down_cat.rows

    @property
    def d_in(self) -> int:
        return self.down_cat.cols

    @property
    def d_out(self) -> int:
        return self.up_cat.rows

    @classmethod
    def empty(cls, d_out: int, d_in: int, precision: str = "single", device=None) -> "ConcatAdapter":
        return cls(
            down_cat=Matrix.zeros(0, d_in, precision, device),
            up_cat=Matrix.zeros(d_out, 0, precision, device),
            provenance=(),
        )

    def validate(self) -> None:
        if self.up_cat.cols != self.down_cat.rows:
            raise DimensionError(
                f"concat rank mismatch: up_cat has {self.up_cat.cols} columns, "
                f"down_cat has {self.down_cat.rows} rows"
            )
        if self.provenance:
            block = self.s / len(self.provenance)
            if block != int(block) or int(block) < 1:
                raise DimensionError("summed rank does not divide into provenance blocks")
        elif self.s != 0:
            raise DimensionError("non-empty concat carries no provenance")


# ---------------------------------------------------------------------------
# Materialised operations (adapters.py:170-258)
# ---------------------------------------------------------------------------


def expert_apply(expert: LoraExpert, x: Matrix, gate_weight: float, recorder: DispatchRecorder) -> Matrix:
    """gate_weight * up @ (down @ x): the unmerged path, exactly two gemm events
    (adapters.py:170-185).  Used by prefill and the baseline strategies only."""
    expert.validate()
    if x.rows != expert.down.cols or x.cols != 1:
        raise DimensionError(f"expert expects a {expert.down.cols}x1 input, got {x.rows}x{x.cols}")
    t = gemm(expert.down, x, recorder, label="adapter")
    u = gemm(expert.up, t, recorder, label="adapter")
    return Matrix(u.data * float(gate_weight), u.precision)


def concat_gated(bank_layer, gate: GateDecision) -> ConcatAdapter:
    """Stack one matrix's chosen experts into a gated block pair (adapters.py:188-211).

    DOWN blocks are scaled by their gate weight in f32 -- the stacked factors are therefore
    "single" even over a bf16 bank -- UP blocks are stacked unscaled.  No events."""
    if len(gate.expert_ids) == 0:
        raise ValueError("gate decision selects no experts")
    experts = []
    for expert_id in gate.expert_ids:
        if not 0 <= expert_id < len(bank_layer):
            raise IndexError(f"expert id {expert_id} outside bank of {len(bank_layer)}")
        experts.append(bank_layer[expert_id])
    down_blocks = [e.down.data.float() * float(w) for e, w in zip(experts, gate.weights)]
    up_blocks = [e.up.data.float() for e in experts]
    return ConcatAdapter(
        down_cat=Matrix(torch.cat(down_blocks, dim=0), "single"),
        up_cat=Matrix(torch.cat(up_blocks, dim=1), "single"),
        provenance=tuple((int(i), float(w), 1) for i, w in zip(gate.expert_ids, gate.weights)),
    )


def build_switch(prev: ConcatAdapter, cur: ConcatAdapter) -> ConcatAdapter:
    """[previous (DOWN negated) | current] in one concat (adapters.py:214-233)."""
    prev.validate()
    cur.validate()
    if prev.d_in != cur.d_in or prev.d_out != cur.d_out:
        raise DimensionError(
            f"switch halves disagree on shape: {prev.d_out}x{prev.d_in} vs {cur.d_out}x{cur.d_in}"
        )
    if prev.down_cat.precision != cur.down_cat.precision:
        raise PrecisionError("switch halves carry mixed precision tags")
    precision = cur.down_cat.precision
    dev = cur.down_cat.data.device
    down = torch.cat([-prev.down_cat.data.to(dev), cur.down_cat.data], dim=0)
    up = torch.cat([prev.up_cat.data.to(dev), cur.up_cat.data], dim=1)
    provenance = tuple((i, w, -sign) for i, w, sign in prev.provenance) + cur.provenance
    return ConcatAdapter(Matrix(down, precision), Matrix(up, precision), provenance)


def merge_all(backbone, concats, sign: int, recorder: DispatchRecorder, tile: TileConfig = DEFAULT_TILE, *, compute: str = "exact") -> None:
    """backbone[l] += sign * up_cat[l] @ down_cat[l] for all l in ONE launch and one sgmm
    event labelled "switch" (adapters.py:236-258)."""
    if len(backbone) != len(concats):
        raise DimensionError(f"{len(backbone)} backbone matrices but {len(concats)} concats")
    table = SegmentTable([Segment(down=c.down_cat, up=c.up_cat, target=f) for f, c in zip(backbone, concats)])
    sgmm(table, sign, recorder, tile=tile, label="switch", compute=compute)


# ---------------------------------------------------------------------------
# The resident form: descriptor table over the expert bank
# ---------------------------------------------------------------------------

_MODES = {"inplace": _capi.AF_SWITCH_INPLACE, "from_pristine": _capi.AF_SWITCH_FROM_PRISTINE}


class SwitchTable:
    """Device-side descriptor table (the GPU form of linalg.py:207-231 `SegmentTable`) over
    every adapted matrix and its slice of the expert bank.  Built once at model load.

    targets[i]  : Matrix d_out x d_in (mutated in place by every switch)
    pristine[i] : Matrix of the same shape, or None for all i
    downs[i]    : tensor [N][r][d_in]   (LoraExpert.down of each expert, adapters.py:53)
    ups[i]      : tensor [N][d_out][r]  (LoraExpert.up,   adapters.py:54)
    """

    def __init__(self, targets, downs, ups, pristine=None):
        if not targets:
            raise DimensionError("segment table is empty")
        if not (len(targets) == len(downs) == len(ups)) or (pristine is not None and len(pristine) != len(targets)):
            raise DimensionError("targets, banks and pristine copies must have one entry per segment")
        descs = []
        tprec = targets[0].precision
        fprec = {torch.bfloat16: "bf16", torch.float32: "single"}.get(downs[0].dtype)
        if fprec is None:
            raise PrecisionError(f"unsupported bank dtype {downs[0].dtype}")
        self.flops_per_rank = 0
        self.factor_elems_per_rank = 0
        self.target_bytes = 0
        for i, (tgt, dn, up) in enumerate(zip(targets, downs, ups)):
            if dn.dim() != 3 or up.dim() != 3:
                raise DimensionError(f"segment {i}: banks must be [N][r][d_in] and [N][d_out][r]")
            n, r, d_in = (int(v) for v in dn.shape)
            if tuple(up.shape) != (n, tgt.rows, r) or d_in != tgt.cols:
                raise DimensionError(
                    f"segment {i}: target is {tgt.rows}x{tgt.cols}, bank blocks are {tuple(up.shape)} / {tuple(dn.shape)}"
                )
            if tgt.precision != tprec or dn.dtype != downs[0].dtype or up.dtype != downs[0].dtype:
                raise PrecisionError("segments of one table carry mixed precision tags")
            if not (tgt.data.is_cuda and dn.is_cuda and up.is_cuda):
                raise DeviceError("operand is not on a CUDA device: the B200 path has no CPU fallback")
            if not (dn.is_contiguous() and up.is_contiguous()):
                raise DimensionError(f"segment {i}: bank tensors must be contiguous")
            pr = pristine[i] if pristine is not None else None
            if pr is not None and (pr.rows != tgt.rows or pr.cols != tgt.cols or pr.precision != tgt.precision):
                raise DimensionError(f"segment {i}: pristine copy does not match its target")
            descs.append(
                _capi.SegmentDesc(
                    target=_ptr(tgt.data), pristine=_ptr(pr.data) if pr is not None else 0,
                    down=_ptr(dn), up=_ptr(up), d_out=tgt.rows, d_in=tgt.cols, rank=r, n_experts=n,
                    ld_target=tgt.cols, ld_down=d_in, ld_up=r, down_expert_stride=r * d_in, up_expert_stride=tgt.rows * r,
                )
            )
            self.flops_per_rank += 2 * tgt.rows * tgt.cols
            self.factor_elems_per_rank += tgt.rows + tgt.cols
            self.target_bytes += tgt.rows * tgt.cols * tgt.itemsize
        self.rank = int(downs[0].shape[1])
        self.n_experts = min(int(d.shape[0]) for d in downs)
        self.factor_itemsize = downs[0].element_size()
        self.device_table = DeviceTable(descs, tprec, fprec, keepalive=(targets, downs, ups, pristine))
        self.n_segments = len(targets)
        self.device = targets[0].data.device
        self._dev_scalar = None

    # -- accounting (identical formulas to linalg.py:293-303) --
    def switch_flops(self, s: int) -> int:
        return self.flops_per_rank * s

    def switch_bytes(self, s: int) -> int:
        return 2 * self.target_bytes + s * self.factor_elems_per_rank * self.factor_itemsize

    def info(self) -> dict:
        return self.device_table.info()

    def status(self) -> None:
        self.device_table.status()

    @staticmethod
    def _split(dec):
        """-> (device pointer or None, host struct or None)"""
        if dec is None:
            return None, None
        if isinstance(dec, DeviceDecision):
            return dec.ptr, None
        if isinstance(dec, GateDecision):
            return None, decision_to_struct(dec)
        raise TypeError(f"decision must be a GateDecision, a DeviceDecision or None, got {type(dec).__name__}")

    def switch(self, prev, cur, *, max_k: int = _capi.AF_MAX_K, scale: float = 1.0, mode: str = "inplace", compute: str = "auto") -> None:
        """W <- W + delta(cur) - delta(prev) on every segment, one launch (model.py:350-357).

        Host decisions (`GateDecision`) are validated before anything moves and raise here
        (IndexError for an expert outside the bank, adapters.py:199-200).  Device decisions
        (`DeviceDecision`) cannot be read without a synchronisation, so the launch is asynchronous:
        the kernel validates, touches nothing when the decision is unusable, and raises into the
        table's status word -- call `status()` (synchronises) at the next point where the host
        waits anyway; `decode_step` / `generate` / `LlamaEngine.decode_step` do."""
        if mode not in _MODES:
            raise ValueError(f"unknown switch mode {mode!r}")
        if compute not in _capi.COMPUTE_MODES:
            raise ValueError(f"unknown compute mode {compute!r}")
        pd, ph = self._split(prev)
        cd, ch = self._split(cur)
        _capi.check(
            _capi.lib().af_fused_switch(
                self.device_table.handle, pd, cd, ph, ch, int(max_k), float(scale), _MODES[mode],
                _capi.COMPUTE_MODES[compute], _capi.stream_ptr(),
            )
        )

    TENSOR_PATH_RANKS = 64   # stacked ranks one mma.sync tensor-path launch holds (include/adafuse_b200.h, af_fused_switch)
    UMMA_PATH_RANKS = 256    # ... and one K-chunked tcgen05 launch (tables of one rank in {8, 16, 32} on 128-multiples)

    def one_launch_ranks(self) -> int:
        """Stacked ranks (blocks x rank) ONE tensor-path launch over this table takes -- the reference's merge is
        one sgmm whatever the stacked rank (adapters.py:236-258); beyond this the engine falls back to passes."""
        if self.info()["umma_path"] and self.rank in (8, 16, 32):
            return self.UMMA_PATH_RANKS
        return self.TENSOR_PATH_RANKS

    def switch_in_passes(self, prev, cur, *, rank: int, max_k: int, scale: float = 1.0, mode: str = "inplace",
                         compute: str = "auto", hold_last: bool = False):
        """The switch of `switch`, for decisions whose stacked rank (blocks x rank) exceeds what one
        tensor-path launch holds (`one_launch_ranks`: 256 on the tcgen05 path, which covers every
        BASELINE configuration in ONE launch; 64 for rank-64 tables and off the tcgen05 path): the
        experts are taken `one_launch_ranks() // rank` at a time -- first the previous decision's (unmerged), then the
        current one's (merged; the first of them from pristine in that mode) -- each pass one
        tensor-path launch over all segments.  The sub-decisions are cut on the device (no host
        round trip, capturable).  Costs one pass over W per launch and rounds W to bf16 once per
        pass instead of once (still fewer roundings than the reference's accumulate-into-target
        order, linalg.py:338-343); the CUDA-core kernel that takes any stacked rank in ONE pass is
        FMA-bound and 5x slower at 256.  Decisions must be DeviceDecisions of exactly max_k experts.
        Returns the number of launches -- or, with hold_last, leaves the last merge pass to the caller
        (who fuses it with the forward, `SegmentGroup.switch_gemv`) and returns its
        (sub-decision, expert count, mode)."""
        for dec in (prev, cur):
            if dec is not None and not isinstance(dec, DeviceDecision):
                raise TypeError("switch_in_passes takes device-resident decisions (DeviceDecision) or None")
        per = max(1, self.one_launch_ranks() // int(rank))
        chunks = [(start, min(per, max_k - start)) for start in range(0, max_k, per)]
        if not hasattr(self, "_sub_decisions"):
            self._sub_decisions = {}
        passes = []
        if mode == "inplace" and prev is not None:
            passes += [("prev", c) for c in chunks]
        if cur is not None:
            passes += [("cur", c) for c in chunks]
        launches = 0
        first_cur = True
        held = None
        for idx, (which, (start, count)) in enumerate(passes):
            src = prev if which == "prev" else cur
            key = (which, start)
            sub = self._sub_decisions.get(key)
            if sub is None or sub.buf.device != src.buf.device:
                sub = self._sub_decisions[key] = DeviceDecision(src.buf.device)
            si, di = src.buf.view(torch.int32), sub.buf.view(torch.int32)
            di[0:1].fill_(count)
            di[1: 1 + count].copy_(si[1 + start: 1 + start + count])                                           # expert ids
            di[1 + _capi.AF_MAX_K: 1 + _capi.AF_MAX_K + count].copy_(si[1 + _capi.AF_MAX_K + start: 1 + _capi.AF_MAX_K + start + count])  # weights (raw bits)
            if which == "prev":
                self.switch(sub, None, max_k=count, scale=scale, compute=compute)
            else:
                pass_mode = mode if (mode == "from_pristine" and first_cur) else "inplace"
                first_cur = False
                if hold_last and idx == len(passes) - 1:
                    held = (sub, count, pass_mode)
                    break
                self.switch(None, sub, max_k=count, scale=scale, compute=compute, mode=pass_mode)
            launches += 1
        if mode == "from_pristine" and cur is None:
            self.refresh()
        return held if hold_last else launches

    def build_plan(self, prev, cur, *, max_k: int = _capi.AF_MAX_K, scale: float = 1.0, mode: str = "inplace") -> None:
        """Once per token: the block list of (prev, cur) for the switch + GEMV launches that pass
        plan_prebuilt=True (adapters.py:188-233 bookkeeping, on the device)."""
        for dec in (prev, cur):
            if dec is not None and not isinstance(dec, DeviceDecision):
                raise TypeError("build_plan takes device-resident decisions (DeviceDecision) or None")
        _capi.check(_capi.lib().af_plan_build(self.device_table.handle, prev.ptr if prev is not None else None,
                                              cur.ptr if cur is not None else None, int(max_k), float(scale), _MODES[mode],
                                              _capi.stream_ptr()))

    def merge(self, dec, **kw) -> None:
        """merge_all(sign=+1) of one decision (adapters.py:236-258)."""
        self.switch(None, dec, **kw)

    def unmerge(self, dec, **kw) -> None:
        """merge_all(sign=-1): model.py:460-474 `finalize_generation` in one launch."""
        self.switch(dec, None, **kw)

    def refresh(self) -> None:
        """model.py:308-312 `_refresh_from_pristine`."""
        _capi.check(_capi.lib().af_refresh_from_pristine(self.device_table.handle, _capi.stream_ptr()))

    def max_deviation(self) -> float:
        """model.py:231-236 `max_backbone_deviation` (synchronises)."""
        if self._dev_scalar is None:
            self._dev_scalar = torch.zeros(1, dtype=torch.float32, device=self.device)
        _capi.check(_capi.lib().af_max_deviation(self.device_table.handle, _ptr(self._dev_scalar), _capi.stream_ptr()))
        return float(self._dev_scalar.item())


# ---------------------------------------------------------------------------
# Serialization (adapters.py:265-306): the reference's npz container, read and written
# ---------------------------------------------------------------------------

_BANK_FORMAT = "lorafuse-bank-v1"


def _load_precision(stored: str, wanted: str | None) -> str:
    """Device precision for arrays stored under the reference's tag: "single"/"double" files load as
    "single" unless the caller asks for "bf16" (values on the bf16 grid survive exactly)."""
    if wanted is not None:
        if wanted not in ("bf16", "single"):
            raise PrecisionError(f"unknown precision tag {wanted!r}")
        return wanted
    return stored if stored in ("bf16", "single") else "single"


def save_bank(bank: ExpertBank, path) -> None:
    """adapters.py:268-284: header + `layer{l}/expert{e}/{down,up}` arrays.  Arrays are written as
    f32 (a bf16 factor upcasts exactly), so the reference's own `load_bank` reads the file; the
    header keeps the device precision tag."""
    import json

    import numpy as np

    bank.validate()
    prec = bank.layers[0][0].down.precision
    header = {"format": _BANK_FORMAT, "n_layers": bank.n_layers, "n_experts": bank.n_experts, "rank": bank.rank,
              "precision": "single" if prec == "bf16" else prec, "device_precision": prec}
    arrays = {"header": np.frombuffer(json.dumps(header).encode("utf-8"), dtype=np.uint8)}
    for li, layer in enumerate(bank.layers):
        for ei, expert in enumerate(layer):
            arrays[f"layer{li}/expert{ei}/down"] = expert.down.numpy().astype(np.float32)
            arrays[f"layer{li}/expert{ei}/up"] = expert.up.numpy().astype(np.float32)
    with open(path, "wb") as fh:
        np.savez(fh, **arrays)


def pack_bank_arrays(archive, n_layers: int, n_experts: int, precision: str, device=None):
    """`layer{l}/expert{e}/{down,up}` arrays -> the packed device layout the switch kernels read:
    per layer one contiguous [N][r][d_in] tensor and one [N][d_out][r] tensor, with an `ExpertBank`
    whose experts are VIEWS into them (no second copy)."""
    import numpy as np

    dtype = PRECISION_DTYPES[precision]
    dev = device if device is not None else default_device()
    bank_down, bank_up, layers = [], [], []
    for li in range(n_layers):
        dn = np.stack([np.asarray(archive[f"layer{li}/expert{ei}/down"], dtype=np.float32) for ei in range(n_experts)])
        up = np.stack([np.asarray(archive[f"layer{li}/expert{ei}/up"], dtype=np.float32) for ei in range(n_experts)])
        dn_t = torch.from_numpy(dn).to(device=dev, dtype=dtype).contiguous()
        up_t = torch.from_numpy(up).to(device=dev, dtype=dtype).contiguous()
        bank_down.append(dn_t)
        bank_up.append(up_t)
        layers.append(tuple(LoraExpert(down=Matrix(dn_t[e], precision), up=Matrix(up_t[e], precision)) for e in range(n_experts)))
    bank = ExpertBank(layers=tuple(layers))
    bank.validate()
    return bank, bank_down, bank_up


def load_bank(path, precision: str | None = None, device=None, packed: bool = False):
    """adapters.py:287-306.  Reads files written by the reference or by `save_bank`.  With
    ``packed=True`` also returns the per-layer packed tensors (`SwitchTable(targets, downs, ups)`)."""
    import json

    import numpy as np

    with np.load(path) as archive:
        header = json.loads(bytes(archive["header"]).decode("utf-8"))
        if header.get("format") != _BANK_FORMAT:
            raise ValueError(f"not a {_BANK_FORMAT} container: {path}")
        prec = _load_precision(header.get("device_precision", header["precision"]), precision)
        bank, downs, ups = pack_bank_arrays(archive, header["n_layers"], header["n_experts"], prec, device)
    return (bank, downs, ups) if packed else bank


class SegmentGroup:
    """Segments of a `SwitchTable` that share one input vector (q|k|v, gate|up, or one matrix):
    the unit of the fused switch + GEMV launch (include/adafuse_b200.h `af_switch_gemv`).  The
    switch of adapters.py:236-258 and the backbone GEMV of model.py:288 over the same weights
    become one pass: every tile is merged, rounded, multiplied with x and written back.

    `seg_ids` may also be a list of lists: a CHAIN of up to four such groups whose inputs depend
    on each other's outputs, run as one launch (`switch_gemv_chain`)."""

    PROLOGUES = {"none": _capi.AF_PRO_NONE, "rmsnorm": _capi.AF_PRO_RMSNORM, "silu_mul": _capi.AF_PRO_SILU_MUL,
                 "rmsnorm_deferred": _capi.AF_PRO_RMSNORM_DEFERRED}

    def __init__(self, table: SwitchTable, seg_ids, cta_share=None):
        """`cta_share` (optional): [n_phases][n_cta] positive floats -- the measured share of each phase's tiles every
        CTA of the launch should get (`af_chain_create_weighted`; `LlamaEngine.calibrate_schedule` produces it)."""
        import ctypes

        seg_ids = list(seg_ids)
        phases = [list(p) for p in seg_ids] if seg_ids and isinstance(seg_ids[0], (list, tuple, range)) else [seg_ids]
        ids = [int(i) for p in phases for i in p]
        arr = (ctypes.c_int32 * max(1, len(ids)))(*ids)
        lens = (ctypes.c_int32 * len(phases))(*[len(p) for p in phases])
        handle = ctypes.c_void_p()
        if cta_share is None:
            _capi.check(_capi.lib().af_chain_create(table.device_table.handle, arr, lens, len(phases), ctypes.byref(handle)))
        else:
            rows = [[float(v) for v in row] for row in cta_share]
            if len(rows) != len(phases) or len({len(r) for r in rows}) != 1:
                raise DimensionError("cta_share must hold one row of per-CTA shares per phase")
            flat = [v for r in rows for v in r]
            share = (ctypes.c_float * len(flat))(*flat)
            _capi.check(_capi.lib().af_chain_create_weighted(table.device_table.handle, arr, lens, len(phases), share, len(rows[0]),
                                                             ctypes.byref(handle)))
        self.handle = handle
        self.table = table  # keeps the af_table (and the tensors it points at) alive
        n_ph, n_units, grid, tiles = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
        x_len, y_rows = (ctypes.c_int32 * 4)(), (ctypes.c_int32 * 4)()
        _capi.check(_capi.lib().af_group_info(handle, ctypes.byref(n_ph), x_len, y_rows, ctypes.byref(n_units), ctypes.byref(grid),
                                              ctypes.byref(tiles)))
        self.n_phases = n_ph.value
        self.x_lens, self.y_rows_all = list(x_len)[: self.n_phases], list(y_rows)[: self.n_phases]
        self.x_len, self.y_rows = self.x_lens[0], self.y_rows_all[0]
        self.n_units, self.grid, self.tiles = n_units.value, grid.value, tiles.value

    def _phase_struct(self, ph: int, acc_out, xin=None, acc_in=None, res=None, h_out=None, prologue="none", norm_w=None, eps: float = 0.0,
                      inv_out=None, inv_in=None):
        if prologue not in self.PROLOGUES:
            raise ValueError(f"unknown prologue {prologue!r}")
        x_len, y_rows = self.x_lens[ph], self.y_rows_all[ph]
        need = x_len * (2 if prologue == "silu_mul" else 1)
        for name, t, dt, n in (("xin", xin, torch.float32, need), ("acc_in", acc_in, torch.int64, need), ("res", res, torch.float32, x_len),
                               ("h_out", h_out, torch.float32, x_len), ("norm_w", norm_w, torch.float32, x_len),
                               ("acc_out", acc_out, torch.int64, y_rows), ("inv_out", inv_out, torch.float32, 1), ("inv_in", inv_in, torch.float32, 1)):
            if t is None:
                continue
            if not t.is_cuda:
                raise DeviceError("operand is not on a CUDA device: the B200 path has no CPU fallback")
            if t.dtype != dt or not t.is_contiguous() or t.numel() < n:
                raise DimensionError(f"{name} must be a contiguous {dt} vector of at least {n} entries")
        p = lambda t: _ptr(t) if t is not None else None  # noqa: E731
        return _capi.GemvPhase(xin=p(xin), acc_in=p(acc_in), res=p(res), h_out=p(h_out), norm_w=p(norm_w), acc_out=p(acc_out),
                               eps=float(eps), prologue=self.PROLOGUES[prologue], inv_out=p(inv_out), inv_in=p(inv_in))

    def switch_gemv_chain(self, prev, cur, phases, phase_done=None, *, max_k: int = _capi.AF_MAX_K, scale: float = 1.0,
                          mode: str = "inplace", pdl: bool = False, plan_prebuilt: bool = False) -> None:
        """One launch over every phase of the chain.  `phases`: one dict per phase with the keyword
        arguments of `switch_gemv` (acc_out, xin | acc_in, res, h_out, prologue, norm_w, eps);
        `phase_done`: int32 tensor of n_phases - 1 zeroed counters."""
        if mode not in _MODES:
            raise ValueError(f"unknown switch mode {mode!r}")
        for dec in (prev, cur):
            if dec is not None and not isinstance(dec, DeviceDecision):
                raise TypeError("the fused switch + GEMV takes device-resident decisions (DeviceDecision) or None")
        if len(phases) != self.n_phases:
            raise DimensionError(f"chain has {self.n_phases} phases, got {len(phases)} descriptions")
        n_counters = self.n_phases - 1 + ((getattr(self, "reduce_mask", 0) >> (self.n_phases - 1)) & 1)
        if n_counters > 0:
            if phase_done is None or phase_done.dtype != torch.int32 or not phase_done.is_cuda or phase_done.numel() < n_counters:
                raise DimensionError(f"phase_done must be a CUDA int32 tensor of {n_counters} zeroed counters")
        structs = (_capi.GemvPhase * self.n_phases)(*[self._phase_struct(i, **ph) for i, ph in enumerate(phases)])
        _capi.check(_capi.lib().af_switch_gemv_chain(
            self.handle, prev.ptr if prev is not None else None, cur.ptr if cur is not None else None, int(max_k), float(scale),
            _MODES[mode], structs, self.n_phases, _ptr(phase_done) if phase_done is not None else None,
            (_capi.AF_CHAIN_PDL if pdl else 0) | (_capi.AF_CHAIN_PLAN_PREBUILT if plan_prebuilt else 0), _capi.stream_ptr()))

    def set_peers(self, peer_offsets, reduce_phases) -> None:
        """Tensor parallelism without a collective between the launches (`af_group_set_peers`; no reference
        counterpart).  `peer_offsets`: byte offsets from this rank's accumulator buffer to every rank's mapping of
        it, this rank included as 0; `reduce_phases`: the row-parallel phases of the chain (o, down) -- their partial
        sums go into EVERY rank's accumulators and the phase is reported on every rank's counter, so the next phase
        starts on the all-reduced vector.  An empty offset list clears the setting."""
        import ctypes

        offs = [int(o) for o in peer_offsets]
        mask = 0
        for ph in reduce_phases:
            if not 0 <= int(ph) < self.n_phases:
                raise ValueError(f"chain has no phase {ph}")
            mask |= 1 << int(ph)
        arr = (ctypes.c_int64 * max(1, len(offs)))(*offs)
        _capi.check(_capi.lib().af_group_set_peers(self.handle, len(offs), arr, mask))
        self.n_peers, self.reduce_mask = len(offs), mask

    def switch_gemv(self, prev, cur, acc_out, *, max_k: int = _capi.AF_MAX_K, scale: float = 1.0, mode: str = "inplace",
                    pdl: bool = False, plan_prebuilt: bool = False, **phase) -> None:
        """acc_out (int64, zeroed by the caller) += fix(W_new . prologue(h)); W <- W_new in place."""
        self.switch_gemv_chain(prev, cur, [dict(acc_out=acc_out, **phase)], None, max_k=max_k, scale=scale, mode=mode, pdl=pdl,
                               plan_prebuilt=plan_prebuilt)

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle:
            _capi.lib().af_group_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def peer_barrier(counter: torch.Tensor, epoch: torch.Tensor, peer_offsets, err_flag: torch.Tensor | None = None) -> None:
    """`af_peer_barrier`: once per token, after this rank zeroed its accumulators and before any rank may push into
    them.  `counter` (int32[1], inside the buffer the peers map) is bumped on every rank and never reset; `epoch`
    (int32[1], private, zero-initialised) counts this rank's barriers on the device, so a captured graph replays."""
    import ctypes

    offs = [int(o) for o in peer_offsets]
    arr = (ctypes.c_int64 * len(offs))(*offs)
    _capi.check(_capi.lib().af_peer_barrier(_ptr(counter), _ptr(epoch), len(offs), arr, _ptr(err_flag) if err_flag is not None else None,
                                            _capi.stream_ptr()))


def peer_wait(counter: torch.Tensor, target: int, err_flag: torch.Tensor | None = None) -> None:
    """`af_peer_wait`: the stream waits until the counter the peers bump has reached `target`."""
    _capi.check(_capi.lib().af_peer_wait(_ptr(counter), int(target), _ptr(err_flag) if err_flag is not None else None, _capi.stream_ptr()))


def peer_bcast(src, slot: torch.Tensor, dst: torch.Tensor, is_root: bool, counter: torch.Tensor, epoch: torch.Tensor, peer_offsets,
               err_flag: torch.Tensor | None = None) -> None:
    """`af_peer_bcast`: the root's record (`src`, same byte size as `dst`) lands in `slot` of every rank and is copied to
    `dst` on every rank -- rank 0's decision of the token, without a library collective."""
    import ctypes

    offs = [int(o) for o in peer_offsets]
    arr = (ctypes.c_int64 * len(offs))(*offs)
    nbytes = dst.numel() * dst.element_size()
    _capi.check(_capi.lib().af_peer_bcast(_ptr(src) if src is not None else None, _ptr(slot), _ptr(dst), nbytes, 1 if is_root else 0,
                                          _ptr(counter), _ptr(epoch), len(offs), arr, _ptr(err_flag) if err_flag is not None else None,
                                          _capi.stream_ptr()))


def peer_argmax(val: torch.Tensor, idx: torch.Tensor, slots: torch.Tensor, my_slot: int, counter: torch.Tensor, epoch: torch.Tensor,
                peer_offsets, out_idx: torch.Tensor, err_flag: torch.Tensor | None = None) -> None:
    """`af_peer_argmax`: every rank's (value, index) pair to every rank; the largest value wins, the lowest index on ties."""
    import ctypes

    offs = [int(o) for o in peer_offsets]
    arr = (ctypes.c_int64 * len(offs))(*offs)
    _capi.check(_capi.lib().af_peer_argmax(_ptr(val), _ptr(idx), _ptr(slots), int(my_slot), _ptr(counter), _ptr(epoch), len(offs), arr,
                                           _ptr(out_idx), _ptr(err_flag) if err_flag is not None else None, _capi.stream_ptr()))
