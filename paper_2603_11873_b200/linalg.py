"""Kernel layer: device matrices, dispatch accounting and the segmented update.

Host-side mirror of /root/reference/pkg/src/lorafuse/linalg.py with the same names, argument
order and error behaviour; every operation is ONE launch of a hand-written sm_100a kernel
through the C ABI (include/adafuse_b200.h) and appends exactly one event to the recorder
(linalg.py:125-159 contract), so `perf`-style accounting keeps working on traces recorded here.

Differences that follow from the device carrier (documented in DESIGN.md):
  * ``Matrix.data`` is a 2-D contiguous ``torch`` tensor; precision tags are ``"bf16"`` (the
    storage type of backbone weights and expert banks on B200) and ``"single"`` (f32:
    activations, gate-folded factors, and the reference's own "single" mode).  ``"double"`` is
    not a device precision here and raises ``PrecisionError`` like any unknown tag
    (linalg.py:58-59).
  * ``gemm`` is the bs=1 decode GEMV (model.py:288, model.py:262): the vector operand is
    always ``"single"``; the matrix operand may be ``"bf16"`` or ``"single"``.
  * A ``Segment`` may pair a ``"bf16"`` target with ``"single"`` factors (gate folding is an
    f32 multiply, adapters.py:202).
There is no CPU fallback: any kernel call on a non-CUDA tensor raises ``DeviceError``.

Attribution: the accounting and table carriers -- ``DispatchEvent``, ``DispatchSummary``,
``DispatchRecorder`` (``record`` / ``mark`` / ``events_since`` / ``counts``), ``TileConfig``, ``Segment`` and
``SegmentTable`` with their validation rules and messages -- are the reference's classes
(linalg.py:110-231) restated: they are the public API this package keeps intact, so names, fields and
error behaviour come from the reference.  ``Matrix`` on a torch tensor, ``DeviceTable`` and every
kernel call are this package's own.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi
from .errors import AliasingError, DeviceError, DimensionError, PrecisionError

# ---------------------------------------------------------------------------
# Matrix
# ---------------------------------------------------------------------------

PRECISION_DTYPES = {"bf16": torch.bfloat16, "single": torch.float32}
_DTYPE_PRECISIONS = {torch.bfloat16: "bf16", torch.float32: "single"}
_AF_DTYPE = {"bf16": _capi.AF_BF16, "single": _capi.AF_F32}


def default_device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")


class Matrix:
    """Dense 2-D row-major array tagged "bf16" or "single" (linalg.py:45-96)."""

    __slots__ = ("data", "precision")

    def __init__(self, data, precision: str | None = None, device=None):
        if isinstance(data, torch.Tensor):
            t = data
        else:
            arr = np.asarray(data)
            if arr.dtype == np.float64 or arr.dtype.kind in "iub":
                arr = arr.astype(np.float32)
            t = torch.from_numpy(np.ascontiguousarray(arr))
        if t.dim() != 2:
            raise DimensionError(f"Matrix requires a 2-D array, got ndim={t.dim()}")
        if precision is None:
            precision = _DTYPE_PRECISIONS.get(t.dtype, "single")
        if precision not in PRECISION_DTYPES:
            raise PrecisionError(f"unknown precision tag {precision!r}")
        if device is None:
            device = t.device if (isinstance(data, torch.Tensor) and t.is_cuda) else default_device()
        self.data = t.to(device=device, dtype=PRECISION_DTYPES[precision]).contiguous()
        self.precision = precision

    @property
    def rows(self) -> int:
        return int(self.data.shape[0])

    @property
    def cols(self) -> int:
        return int(self.data.shape[1])

    @property
    def itemsize(self) -> int:
        return int(self.data.element_size())

    @classmethod
    def zeros(cls, rows: int, cols: int, precision: str = "bf16", device=None) -> "Matrix":
        if rows < 0 or cols < 0:
            raise DimensionError("matrix dimensions must be non-negative")
        if precision not in PRECISION_DTYPES:
            raise PrecisionError(f"unknown precision tag {precision!r}")
        dev = device if device is not None else default_device()
        return cls(torch.zeros((rows, cols), dtype=PRECISION_DTYPES[precision], device=dev), precision)

    @classmethod
    def identity(cls, n: int, precision: str = "bf16", device=None) -> "Matrix":
        dev = device if device is not None else default_device()
        return cls(torch.eye(n, dtype=PRECISION_DTYPES[precision], device=dev), precision)

    def copy(self) -> "Matrix":
        return Matrix(self.data.clone(), self.precision)

    def is_finite(self) -> bool:
        return bool(torch.isfinite(self.data.float()).all().item())

    def numpy(self) -> np.ndarray:
        """Host copy as float32 (bf16 values widen exactly)."""
        return self.data.detach().float().cpu().numpy()

    def bits(self) -> np.ndarray:
        """Host copy of the raw bf16 bit patterns (uint16); bf16 matrices only."""
        if self.precision != "bf16":
            raise PrecisionError("bits() is defined for bf16 matrices")
        return self.data.detach().view(torch.int16).cpu().numpy().view(np.uint16)

    def __repr__(self) -> str:  # pragma: no cover - debug aid
        return f"Matrix({self.rows}x{self.cols}, {self.precision}, {self.data.device})"


def _require_cuda(*mats: Matrix) -> None:
    for m in mats:
        if not m.data.is_cuda:
            raise DeviceError("operand is not on a CUDA device: the B200 path has no CPU fallback")


def _ptr(t: torch.Tensor) -> int:
    return int(t.data_ptr()) if t.numel() else 0


# ---------------------------------------------------------------------------
# Dispatch recording (linalg.py:99-159)
# ---------------------------------------------------------------------------

EVENT_KINDS = ("gemm", "sgmm", "elementwise", "reduce")


@dataclass(frozen=True, slots=True)
class DispatchEvent:
    """One device launch."""

    kind: str
    flops: int
    bytes_touched: int
    label: str = "other"


@dataclass(frozen=True, slots=True)
class DispatchSummary:
    counts: dict
    total_flops: int
    total_bytes: int


class DispatchRecorder:
    """Append-only event log; one recorder per engine, never shared."""

    def __init__(self):
        self.events: list[DispatchEvent] = []

    def record(self, kind: str, flops: int, bytes_touched: int, label: str = "other") -> None:
        if kind not in EVENT_KINDS:
            raise ValueError(f"unknown event kind {kind!r}")
        if flops < 0 or bytes_touched < 0:
            raise ValueError("flops and bytes_touched must be non-negative")
        self.events.append(DispatchEvent(kind, int(flops), int(bytes_touched), label))

    def mark(self) -> int:
        return len(self.events)

    def events_since(self, mark: int) -> list[DispatchEvent]:
        return self.events[mark:]

    def counts(self) -> dict:
        out = dict.fromkeys(EVENT_KINDS, 0)
        for ev in self.events:
            out[ev.kind] += 1
        return out

    def reset_and_report(self) -> DispatchSummary:
        summary = DispatchSummary(
            counts=self.counts(),
            total_flops=sum(ev.flops for ev in self.events),
            total_bytes=sum(ev.bytes_touched for ev in self.events),
        )
        self.events.clear()
        return summary


# ---------------------------------------------------------------------------
# Segments and tiles (linalg.py:162-231)
# ---------------------------------------------------------------------------


@dataclass(frozen=True, slots=True)
class TileConfig:
    """Tile extents of the reference's loop nest (linalg.py:167-180).  Results are
    bit-identical for every TileConfig there; here the argument is accepted and ignored --
    the device kernels pick their own tiles and keep the same ascending-rank order."""

    m: int = 32
    n: int = 32
    k: int = 8

    def __post_init__(self):
        if self.m < 1 or self.n < 1 or self.k < 1:
            raise ValueError(f"tile extents must be positive, got {self}")


DEFAULT_TILE = TileConfig()


@dataclass(slots=True)
class Segment:
    """target += sign * up @ down; down is s x d_in, up is d_out x s (linalg.py:183-205)."""

    down: Matrix
    up: Matrix
    target: Matrix

    @property
    def rank_total(self) -> int:
        return self.down.rows

    def validate(self) -> None:
        if self.up.cols != self.down.rows:
            raise DimensionError(
                f"segment rank mismatch: up has {self.up.cols} columns, down has {self.down.rows} rows"
            )
        if self.up.rows != self.target.rows or self.down.cols != self.target.cols:
            raise DimensionError(
                f"segment target is {self.target.rows}x{self.target.cols}, "
                f"update is {self.up.rows}x{self.down.cols}"
            )
        if self.up.precision != self.down.precision:
            raise PrecisionError("segment factors carry mixed precision tags")
        if self.target.precision != self.up.precision and not (
            self.target.precision == "bf16" and self.up.precision == "single"
        ):
            raise PrecisionError("segment operands carry mixed precision tags")


@dataclass(slots=True)
class SegmentTable:
    """Non-empty list of segments with pairwise distinct targets (linalg.py:207-231)."""

    segments: list = field(default_factory=list)

    def validate(self) -> None:
        if not self.segments:
            raise DimensionError("segment table is empty")
        seen = set()
        first = self.segments[0]
        for seg in self.segments:
            seg.validate()
            if seg.target.precision != first.target.precision or seg.up.precision != first.up.precision:
                raise PrecisionError("segments of one table carry mixed precision tags")
            key = seg.target.data.data_ptr() if seg.target.data.numel() else id(seg.target.data)
            if key in seen:
                raise AliasingError("two segments share one target matrix")
            seen.add(key)

    def __len__(self) -> int:
        return len(self.segments)


class DeviceTable:
    """Owner of one `af_table` (the device-side descriptor table + TMA maps)."""

    def __init__(self, descs: list, target_precision: str, factor_precision: str, keepalive=()):
        arr = (_capi.SegmentDesc * len(descs))(*descs)
        handle = ctypes.c_void_p()
        _capi.check(
            _capi.lib().af_table_create(
                arr, len(descs), _AF_DTYPE[target_precision], _AF_DTYPE[factor_precision], ctypes.byref(handle)
            )
        )
        self.handle = handle
        self.n_segments = len(descs)
        self._keepalive = keepalive  # tensors whose addresses the table holds

    def info(self) -> dict:
        n, elems, units, fast = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        _capi.check(
            _capi.lib().af_table_info(self.handle, ctypes.byref(n), ctypes.byref(elems), ctypes.byref(units), ctypes.byref(fast))
        )
        return {
            "n_segments": n.value,
            "target_elems": elems.value,
            "n_units": units.value,
            "tma_path": bool(fast.value & 1),
            "tensor_path": bool(fast.value & 2),
            "umma_path": bool(fast.value & 4),
        }

    def status(self) -> None:
        """Raise what a kernel flagged for a device-resident decision (synchronises)."""
        _capi.check(_capi.lib().af_table_status(self.handle, _capi.stream_ptr()))

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle:
            _capi.lib().af_table_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def _materialised_desc(seg: Segment) -> _capi.SegmentDesc:
    s = seg.rank_total
    return _capi.SegmentDesc(
        target=_ptr(seg.target.data),
        pristine=0,
        down=_ptr(seg.down.data),
        up=_ptr(seg.up.data),
        d_out=seg.target.rows,
        d_in=seg.target.cols,
        rank=s,
        n_experts=1,
        ld_target=seg.target.cols,
        ld_down=seg.down.cols,
        ld_up=max(s, 0),
        down_expert_stride=0,
        up_expert_stride=0,
    )


# ---------------------------------------------------------------------------
# Kernels
# ---------------------------------------------------------------------------


def _check_pair(a: Matrix, b: Matrix) -> None:
    if a.cols != b.rows:
        raise DimensionError(f"inner dimensions differ: {a.rows}x{a.cols} @ {b.rows}x{b.cols}")


def gemm(a: Matrix, b: Matrix, recorder: DispatchRecorder, label: str = "other", *, epilogue: str = "none", residual: Matrix | None = None) -> Matrix:
    """C = A @ B as one launch and one gemm event (linalg.py:246-259).

    The decode path only ever multiplies by one vector: ``A (m x k) @ x (k x 1)`` runs the
    row-major GEMV kernel, ``x^T (1 x k) @ B (k x n)`` (model.py:262 `_unembed`) the transposed
    one.  The vector side must be "single".  ``epilogue="gelu_residual"`` fuses
    model.py:298-305 (``residual + gelu(y)``) into the same launch.
    """
    _check_pair(a, b)
    lib = _capi.lib()
    st = None
    if b.cols == 1:
        if b.precision != "single":
            raise PrecisionError(f"precision mismatch: the vector operand must be single, got {b.precision}")
        _require_cuda(a, b)
        st = _capi.stream_ptr()
        out = torch.empty((a.rows, 1), dtype=torch.float32, device=a.data.device)
        epi = {"none": _capi.AF_EPI_NONE, "gelu_residual": _capi.AF_EPI_GELU_RESIDUAL, "residual": _capi.AF_EPI_RESIDUAL}.get(epilogue)
        if epi is None:
            raise ValueError(f"unknown epilogue {epilogue!r}")
        res_ptr = 0
        if epi != _capi.AF_EPI_NONE:
            if residual is None or residual.rows != a.rows or residual.cols != 1 or residual.precision != "single":
                raise DimensionError("epilogue needs a single-precision residual of the output shape")
            res_ptr = _ptr(residual.data)
        _capi.check(
            lib.af_gemv(_ptr(a.data), _AF_DTYPE[a.precision], a.rows, a.cols, a.cols, _ptr(b.data), _ptr(out), epi, res_ptr, st)
        )
    elif a.rows == 1:
        if a.precision != "single":
            raise PrecisionError(f"precision mismatch: the vector operand must be single, got {a.precision}")
        if epilogue != "none":
            raise ValueError("epilogues are defined for the column-vector GEMV only")
        _require_cuda(a, b)
        st = _capi.stream_ptr()
        out = torch.empty((1, b.cols), dtype=torch.float32, device=b.data.device)
        _capi.check(lib.af_gemv_t(_ptr(b.data), _AF_DTYPE[b.precision], b.rows, b.cols, b.cols, _ptr(a.data), _ptr(out), st))
    else:
        raise DimensionError(
            f"the B200 decode path multiplies by one vector (bs=1); got {a.rows}x{a.cols} @ {b.rows}x{b.cols}"
        )
    recorder.record(
        "gemm",
        flops=2 * a.rows * a.cols * b.cols,
        bytes_touched=a.rows * a.cols * a.itemsize + b.rows * b.cols * b.itemsize + a.rows * b.cols * 4,
        label=label,
    )
    return Matrix(out, "single")


def _table_flops(table: SegmentTable) -> int:
    return sum(2 * s.up.rows * s.rank_total * s.down.cols for s in table.segments)


def _table_bytes(table: SegmentTable) -> int:
    total = 0
    for s in table.segments:
        total += s.up.rows * s.up.cols * s.up.itemsize + s.down.rows * s.down.cols * s.down.itemsize
        total += 2 * s.target.rows * s.target.cols * s.target.itemsize
    return total


def _launch_sgmm(table: SegmentTable, sign: int, compute: str) -> None:
    for seg in table.segments:
        _require_cuda(seg.down, seg.up, seg.target)
    first = table.segments[0]
    descs = [_materialised_desc(seg) for seg in table.segments]
    dev = DeviceTable(descs, first.target.precision, first.up.precision)
    try:
        _capi.check(_capi.lib().af_sgmm(dev.handle, int(sign), _capi.COMPUTE_MODES[compute], _capi.stream_ptr()))
        torch.cuda.current_stream().synchronize()  # the table (and its maps) die with this call
    finally:
        dev.close()


def gemm_accumulate_inplace(c: Matrix, a: Matrix, b: Matrix, sign: int, recorder: DispatchRecorder, label: str = "other") -> None:
    """C += sign * A @ B in one launch, one gemm event (linalg.py:262-290): the product is
    accumulated from zero in f32 and added to C once."""
    if sign not in (1, -1):
        raise ValueError(f"sign must be +1 or -1, got {sign}")
    _check_pair(a, b)
    if c.rows != a.rows or c.cols != b.cols:
        raise DimensionError(f"accumulate target is {c.rows}x{c.cols}, product is {a.rows}x{b.cols}")
    seg = Segment(down=b, up=a, target=c)
    seg.validate()
    if c.rows and c.cols:
        _launch_sgmm(SegmentTable([seg]), sign, "fma")
    recorder.record(
        "gemm",
        flops=2 * a.rows * a.cols * b.cols,
        bytes_touched=a.rows * a.cols * a.itemsize + b.rows * b.cols * b.itemsize + 2 * c.rows * c.cols * c.itemsize,
        label=label,
    )


def sgmm(table: SegmentTable, sign: int, recorder: DispatchRecorder, tile: TileConfig = DEFAULT_TILE, label: str = "other", *, compute: str = "exact") -> None:
    """Apply every segment's update in ONE launch and ONE sgmm event (linalg.py:306-346).

    ``compute="exact"`` (default) keeps the reference's arithmetic bit for bit: per element a
    strict ascending-rank sequence of (multiply, round)(add, round) into the target value,
    rounded to the target's storage type once at the end.  ``"fma"`` / ``"mma"`` / ``"auto"``
    are the fast orders (within 1 bf16 ulp of it).  ``tile`` is accepted for signature parity.
    """
    if sign not in (1, -1):
        raise ValueError(f"sign must be +1 or -1, got {sign}")
    if compute not in _capi.COMPUTE_MODES:
        raise ValueError(f"unknown compute mode {compute!r}")
    table.validate()
    _launch_sgmm(table, sign, compute)
    recorder.record("sgmm", flops=_table_flops(table), bytes_touched=_table_bytes(table), label=label)


def sgmm_sequential(table: SegmentTable, sign: int, recorder: DispatchRecorder, label: str = "other") -> None:
    """Same updates, one launch and one gemm event per segment (linalg.py:349-358)."""
    table.validate()
    for seg in table.segments:
        gemm_accumulate_inplace(seg.target, seg.up, seg.down, sign, recorder, label=label)
