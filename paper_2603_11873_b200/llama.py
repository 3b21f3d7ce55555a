"""Llama-shaped AdaFuse decode engine (BASELINE.json configs 2-5).

The reference's decoder has one adapted d x d matrix per layer (model.py:3-7); the
configurations the headline metric is quoted on adapt q/k/v/o/gate/up/down of a Llama block.
This module is the same per-token hot path -- model.py:332-371 `_merged_pass`:

    pre-gate once per token on the embedding row  ->  ONE fused switch over all 7 x L
    adapted matrices  ->  plain backbone GEMVs  ->  lm_head  ->  argmax

on those shapes.  Everything per token stays on the device and is a fixed launch sequence,
so a whole step is captured once in a CUDA graph and replayed.

Tensor parallelism: q/k/v/gate/up are column-parallel (d_out split), o/down
row-parallel (d_in split); each rank builds the descriptor table over ITS shard and runs the
identical switch kernel -- no data-path collective in the switch; the routing decision is
computed on rank 0 and broadcast (one 128-byte NCCL broadcast per token).  The decode GEMVs
need the usual two all-reduces per layer and an (value, index) all-gather for the
vocab-parallel lm_head.
"""

from __future__ import annotations

import math
import os
import zlib
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _capi
from .adapters import SegmentGroup, SwitchTable
from .errors import ConfigError, DimensionError, InputError, StateError
from .linalg import DispatchRecorder, Matrix, _ptr
from .routing import DECISION_BYTES, DeviceDecision, GateDecision

SEGMENT_NAMES = ("q", "k", "v", "o", "gate", "up", "down")
_COLUMN_PARALLEL = ("q", "k", "v", "gate", "up")


@dataclass(frozen=True, slots=True)
class LlamaConfig:
    layers: int = 2
    hidden: int = 256
    ffn: int = 512
    n_heads: int = 4
    n_kv_heads: int = 2
    vocab: int = 512
    experts: int = 8
    rank: int = 8
    top_k: int = 2
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    max_seq: int = 256
    seed: int = 0
    tp_size: int = 1
    tp_rank: int = 0
    compute: str = "auto"
    switch_mode: str = "inplace"     # or "from_pristine"
    # model.py:344-349: every `refresh_every` decoded tokens the live weights are rebuilt from the pristine copy
    # (bf16 storage re-rounds W at every in-place switch, a ~0.3 sqrt(T) ulp random walk the f32 reference does
    # not have; 16 keeps the logits within 1e-2 of the reference's trajectory).  Here the refresh costs nothing:
    # "copy W0, then merge the current decision" IS the from-pristine switch, so the refreshing token's one
    # launch reads W0 instead of W -- same bytes, no extra pass.  0 = never; needs keep_pristine.
    refresh_every: int = 16
    adapters: bool = True            # False = adapter-free backbone (the reference's BASE strategy)
    keep_pristine: bool = True
    attn_splits: int = 0             # CTAs per head in decode attention; 0 = auto (one per 64 positions of max_seq, at most 32)
    # "chase": the forward GEMV of every projection is fused into the switch of its weights (one pass
    # over W per token instead of switch + forward); "separate": one switch launch, then plain GEMVs;
    # "auto": chase when it applies (adapters, single rank, tensor path)
    forward_mode: str = "auto"
    chain: bool = True               # chase: o -> gate|up -> down -> next q|k|v as ONE launch with in-kernel phase barriers
    split_switch: bool = True        # > 64 stacked ranks: several tensor-path passes instead of one CUDA-core pass
    defer_norm: bool = True          # chase on the tcgen05 path: RMSNorm scales computed by one CTA, applied by the consumers
    # Tensor parallelism: True = the row-parallel projections (o, down) push their fixed-point partial sums into every
    # rank's accumulators from the GEMV epilogue (peer memory over NVLink; `PeerBuffer`), so the chained launch carries
    # to TP and no collective sits between the launches of a layer; False = one NCCL all-reduce after o and after down;
    # None = push when tp_size > 1, the tcgen05 path applies and the ranks can map each other's buffer (env AF_TP_PUSH=0: never)
    tp_push: bool | None = None
    gemv_chain: bool = True          # plain forward (separate / adapter-free): the same four projections as one persistent GEMV launch
    # ... and the whole forward of a token -- attention included -- as ONE launch over a device-side phase table
    # (af_forward_persistent).  Correct and tested, but OFF: measured on Llama-2-7B at 1024 positions the adapter-free
    # decode is 3.51 ms per token against 2.82 ms for one chained launch per layer + the attention kernel -- inside one
    # launch the attention is two more phases, and a phase boundary (grid barrier + input vector + pipeline restart
    # ~ 4-5 us) costs as much as the programmatic-dependent-launch hand-over it replaces (~14 us per layer for three).
    persistent_forward: bool = False
    # chained chase launches: time every CTA's phases once at engine build and split each phase's tiles by the measured
    # rates (`calibrate_schedule`).  Off: measured on Llama-2-7B, the spread of the CTAs' arrival at a phase barrier
    # (~4 us) is tile granularity (+-1 tile of 1.6 us) and unit changes, not a per-SM rate -- recalibrating moves it to
    # other CTAs without shrinking it (5.50 ms per token either way).
    calibrate: bool = False

    def validate(self) -> None:
        for name in ("layers", "hidden", "ffn", "n_heads", "n_kv_heads", "vocab", "experts", "rank", "top_k", "max_seq", "tp_size"):
            v = getattr(self, name)
            if not isinstance(v, int) or isinstance(v, bool) or v < 1:
                raise ValueError(f"{name} must be a positive integer, got {v!r}")
        if self.hidden % self.n_heads or self.n_heads % self.n_kv_heads:
            raise ValueError("hidden must divide into heads, heads into kv heads")
        if (self.hidden // self.n_heads) % 2 or self.hidden // self.n_heads > 256:
            raise ValueError("head_dim must be even and <= 256")
        if self.top_k > self.experts or self.top_k > _capi.AF_MAX_K:
            raise ValueError(f"top_k={self.top_k} exceeds experts={self.experts} or {_capi.AF_MAX_K}")
        if self.rank > self.hidden:
            raise ValueError(f"rank={self.rank} exceeds hidden={self.hidden}")
        if not 0 <= self.tp_rank < self.tp_size:
            raise ValueError("tp_rank outside [0, tp_size)")
        if self.n_kv_heads % self.tp_size or self.ffn % self.tp_size or self.vocab % self.tp_size:
            raise ValueError("kv heads, ffn and vocab must divide by tp_size")
        if (self.ffn // self.tp_size) % 8 or self.hidden % 8:
            raise ValueError("hidden and the local ffn width must be multiples of 8 (16-byte bf16 rows)")
        if self.compute not in _capi.COMPUTE_MODES:
            raise ValueError(f"unknown compute mode {self.compute!r}")
        if self.switch_mode not in ("inplace", "from_pristine"):
            raise ValueError(f"unknown switch mode {self.switch_mode!r}")
        if self.switch_mode == "from_pristine" and not self.keep_pristine:
            raise ValueError("from_pristine needs keep_pristine")
        if not isinstance(self.refresh_every, int) or isinstance(self.refresh_every, bool) or self.refresh_every < 0:
            raise ValueError(f"refresh_every must be a non-negative integer, got {self.refresh_every!r}")
        if self.forward_mode not in ("auto", "chase", "separate"):
            raise ValueError(f"unknown forward mode {self.forward_mode!r}")
        if self.forward_mode == "chase" and not self.adapters:
            raise ValueError("forward_mode='chase' needs adapters")

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads

    def segment_shapes(self) -> dict:
        """Local (per-rank) d_out x d_in of the seven adapted matrices of one layer."""
        d, hd, tp = self.hidden, self.head_dim, self.tp_size
        q, kv, f = self.n_heads // tp * hd, self.n_kv_heads // tp * hd, self.ffn // tp
        return {"q": (q, d), "k": (kv, d), "v": (kv, d), "o": (d, q), "gate": (f, d), "up": (f, d), "down": (d, f)}

    def full_segment_shapes(self) -> dict:
        return replace(self, tp_size=1, tp_rank=0).segment_shapes()

    def switch_bytes(self, steady: bool = True) -> int:
        """Algorithmic bytes of one switch on this rank."""
        s = (2 if steady and self.switch_mode == "inplace" else 1) * self.top_k * self.rank
        return self.layers * sum(4 * o * i + 2 * s * (o + i) for o, i in self.segment_shapes().values())

    def decode_bytes(self) -> int:
        """Bytes one decode forward must read on this rank: every W once + lm_head."""
        w = self.layers * sum(2 * o * i for o, i in self.segment_shapes().values())
        return w + 2 * (self.vocab // self.tp_size) * self.hidden


PRESETS = {
    # BASELINE.json configs[1..4]
    "llama2-7b": dict(layers=32, hidden=4096, ffn=11008, n_heads=32, n_kv_heads=32, vocab=32000, experts=8, rank=8, top_k=2),
    "llama3-8b": dict(layers=32, hidden=4096, ffn=14336, n_heads=32, n_kv_heads=8, vocab=128256, experts=16, rank=16, top_k=2,
                      rope_theta=500000.0),
    "llama2-13b": dict(layers=40, hidden=5120, ffn=13824, n_heads=40, n_kv_heads=40, vocab=32000, experts=8, rank=8, top_k=2),
    "llama2-70b": dict(layers=80, hidden=8192, ffn=28672, n_heads=64, n_kv_heads=8, vocab=32000, experts=8, rank=32, top_k=4),
    "tiny": dict(layers=2, hidden=256, ffn=512, n_heads=4, n_kv_heads=2, vocab=512, experts=8, rank=8, top_k=2),
}


def preset(name: str, **overrides) -> LlamaConfig:
    if name not in PRESETS:
        raise ConfigError(f"unknown preset {name!r}; known: {sorted(PRESETS)}")
    cfg = LlamaConfig(**{**PRESETS[name], **overrides})
    cfg.validate()
    return cfg


# ---------------------------------------------------------------------------
# Synthetic weights
# ---------------------------------------------------------------------------


def tensor_seed(seed: int, name: str) -> int:
    return (zlib.crc32(name.encode()) ^ (seed * 0x9E3779B1)) & 0xFFFFFFFF


def host_tensor(cfg: LlamaConfig, name: str, shape, fan_in: int) -> np.ndarray:
    """Full (unsharded) tensor `name`: PCG64(seed ^ crc(name)), uniform +-1/sqrt(fan_in)
    (the reference's distribution, model.py:184-189), drawn in f64, cast to f32.  Keyed by
    NAME so any rank -- and the CPU oracle -- regenerates exactly the slice it needs."""
    rng = np.random.Generator(np.random.PCG64(tensor_seed(cfg.seed, name)))
    b = 1.0 / math.sqrt(fan_in)
    return rng.uniform(-b, b, size=shape).astype(np.float32)


def shard_rows(a, tp, rank):
    n = a.shape[-2] // tp
    return a[..., rank * n:(rank + 1) * n, :]


def shard_cols(a, tp, rank):
    n = a.shape[-1] // tp
    return a[..., rank * n:(rank + 1) * n]


def host_weights(cfg: LlamaConfig) -> dict:
    """All weights of THIS rank as f32 host arrays (small configs / parity runs)."""
    full = cfg.full_segment_shapes()
    tp, rk = cfg.tp_size, cfg.tp_rank
    hd = cfg.head_dim
    out = {
        "embed": host_tensor(cfg, "embed", (cfg.vocab, cfg.hidden), cfg.hidden),
        "router": host_tensor(cfg, "router", (cfg.experts, cfg.hidden), cfg.hidden),
        "lm_head": shard_rows(host_tensor(cfg, "lm_head", (cfg.vocab, cfg.hidden), cfg.hidden), tp, rk),
        "final_norm": 1.0 + 0.1 * host_tensor(cfg, "final_norm", (cfg.hidden,), 1),
        "layers": [],
    }
    for li in range(cfg.layers):
        lw = {"attn_norm": 1.0 + 0.1 * host_tensor(cfg, f"l{li}.attn_norm", (cfg.hidden,), 1),
              "ffn_norm": 1.0 + 0.1 * host_tensor(cfg, f"l{li}.ffn_norm", (cfg.hidden,), 1)}
        for name in SEGMENT_NAMES:
            d_out, d_in = full[name]
            w = host_tensor(cfg, f"l{li}.{name}.w", (d_out, d_in), d_in)
            dn = host_tensor(cfg, f"l{li}.{name}.down", (cfg.experts, cfg.rank, d_in), d_in)
            up = host_tensor(cfg, f"l{li}.{name}.up", (cfg.experts, d_out, cfg.rank), cfg.rank)
            if name in _COLUMN_PARALLEL:   # split d_out: shard W rows and UP rows, replicate DOWN
                w, up = shard_rows(w, tp, rk), shard_rows(up, tp, rk)
            else:                          # split d_in: shard W cols and DOWN cols, replicate UP
                w, dn = shard_cols(w, tp, rk), shard_cols(dn, tp, rk)
            lw[name] = {"w": np.ascontiguousarray(w), "down": np.ascontiguousarray(dn), "up": np.ascontiguousarray(up)}
        out["layers"].append(lw)
    _ = hd
    return out


def rope_tables(cfg: LlamaConfig):
    half = cfg.head_dim // 2
    inv = cfg.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim)
    ang = np.arange(cfg.max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


# ---------------------------------------------------------------------------
# Collectives (only where the path has a real exchange)
# ---------------------------------------------------------------------------


class PeerBuffer:
    """int64 words of device memory that every tensor-parallel rank maps (`include/adafuse_b200.h`, af_group_set_peers):
    `tensor` is this rank's region, `offsets[w]` the byte distance from it to rank w's region as THIS process sees it
    (own rank: 0).  The engine puts its fixed-point accumulators, phase counters and the token barrier's counter there."""

    def __init__(self, tensor: torch.Tensor, offsets, keep=None):
        if tensor.dtype != torch.int64 or not tensor.is_contiguous():
            raise DimensionError("a peer buffer is a contiguous int64 tensor")
        self.tensor, self.offsets, self._keep = tensor, [int(o) for o in offsets], keep
        if self.offsets.count(0) != 1:
            raise ValueError("peer offsets must contain this rank (0) exactly once")

    @classmethod
    def local(cls, n_words: int, device) -> "PeerBuffer":
        """A single rank: the only peer is the rank itself (tests; the same kernels and counters run)."""
        return cls(torch.zeros(n_words, dtype=torch.int64, device=device), [0])

    @classmethod
    def symmetric(cls, n_words: int, device, group=None) -> "PeerBuffer":
        """One buffer per rank of `group`, mapped by every other rank through torch symmetric memory (CUDA VMM / NVLink
        peer access).  A collective call: every rank of the group makes it with the same size."""
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        t = symm.empty(n_words, dtype=torch.int64, device=device)
        t.zero_()
        hdl = symm.rendezvous(t, group if group is not None else dist.group.WORLD)
        ptrs = [int(p) for p in hdl.buffer_ptrs]
        torch.cuda.synchronize(device)
        dist.barrier(group=group)                      # every region is zeroed before anybody pushes into it
        return cls(t, [p - ptrs[hdl.rank] for p in ptrs], keep=hdl)

    @classmethod
    def ipc(cls, n_words: int, device, group=None) -> "PeerBuffer":
        """One buffer per rank of `group`, mapped by the other ranks through CUDA IPC handles exchanged over the process
        group (any backend): the ranks of one node -- on different GPUs with peer access, or, for tests, on the SAME
        GPU, which torch symmetric memory refuses.  A collective call."""
        import torch.distributed as dist

        t = torch.zeros(n_words, dtype=torch.int64, device=device)
        meta = t.untyped_storage()._share_cuda_()          # cudaIpcGetMemHandle of the block + this storage's offset in it
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        metas = [None] * world
        dist.all_gather_object(metas, meta, group=group)
        views, offsets = [], []
        for w, m in enumerate(metas):
            if w == rank:
                offsets.append(0)
                continue
            storage = torch.UntypedStorage._new_shared_cuda(*m)     # cudaIpcOpenMemHandle (peer access enabled lazily)
            view = torch.empty(0, dtype=torch.int64, device=device).set_(storage)
            views.append(view)
            offsets.append(view.data_ptr() - t.data_ptr())
        torch.cuda.synchronize(device)
        dist.barrier(group=group)                          # every region exists, is zeroed and is mapped everywhere
        return cls(t, offsets, keep=views)


class Collectives:
    """torch.distributed plumbing of the TP path.  With tp_size == 1 every method is a no-op."""

    def __init__(self, group=None, tp_size: int = 1):
        self.group = group
        self.tp_size = tp_size
        if tp_size > 1:
            import torch.distributed as dist

            if not dist.is_initialized():
                raise StateError("tp_size > 1 needs torch.distributed to be initialised")
            self.dist = dist

    def broadcast_decision(self, buf: torch.Tensor) -> None:
        """The ONLY collective of the switch path: rank 0's 128-byte decision record."""
        if self.tp_size > 1:
            self.dist.broadcast(buf, src=self.dist.get_global_rank(self.group, 0) if self.group is not None else 0, group=self.group)

    def all_reduce_sum(self, t: torch.Tensor) -> None:
        if self.tp_size > 1:
            self.dist.all_reduce(t, group=self.group)

    def argmax_pairs(self, val: torch.Tensor, idx: torch.Tensor, out_idx: torch.Tensor) -> None:
        """Vocab-parallel argmax: gather (value, index) pairs, keep the largest value, lowest
        index on ties (model.py:396)."""
        if self.tp_size == 1:
            return
        pair = torch.stack([val.view(1), idx.view(1).to(torch.float32)], dim=1)  # idx < 2^24 is exact in f32
        gathered = [torch.empty_like(pair) for _ in range(self.dist.get_world_size(self.group))]
        self.dist.all_gather(gathered, pair, group=self.group)
        allp = torch.cat(gathered, dim=0)
        best = torch.max(allp[:, 0])
        cand = torch.where(allp[:, 0] == best, allp[:, 1], torch.full_like(allp[:, 1], float("inf")))
        out_idx.copy_(torch.min(cand).to(torch.int32).view(1))


class NoPeers(Collectives):
    """Exchange layer of a shard inspected in isolation (switch-only use: nothing to exchange)."""

    def __init__(self):
        self.group, self.tp_size = None, 1


# ---------------------------------------------------------------------------
# Engine
# ---------------------------------------------------------------------------


def _on_device(fn):
    """Run a public engine method with the engine's device current: the C ABI launches on the current
    device's stream and configures kernels per device, so an engine built on cuda:1 must not be
    driven while cuda:0 is current."""
    import functools

    @functools.wraps(fn)
    def wrapper(self, *a, **kw):
        if torch.cuda.current_device() == self.dev.index:
            return fn(self, *a, **kw)
        with torch.cuda.device(self.dev):
            return fn(self, *a, **kw)

    return wrapper


PEER_TAIL_WORDS = 32     # int64 words behind the accumulator arena in a PeerBuffer: counters, decision slot, argmax slots


class PeerCollectives:
    """The exchanges of a tp_push step that are not sums, over the ranks' peer mappings instead of a library collective
    (`af_peer_bcast`, `af_peer_argmax`): rank 0's decision record and the vocab-parallel argmax.  With the all-reduces
    pushed from the GEMV epilogues this leaves a tensor-parallel token without any NCCL call.  Layout of the tail
    (int64 words): 0 = barrier | bcast counters (int32 each), 1 = gather counter, 2..17 = decision slot, 18..25 = pairs."""

    def __init__(self, tail: torch.Tensor, offsets, rank: int, err_flag: torch.Tensor):
        if tail.numel() < PEER_TAIL_WORDS:
            raise DimensionError("the peer buffer's tail is too small")
        c32 = tail[:2].view(torch.int32)
        self.barrier_counter, self.bcast_counter, self.gather_counter = c32[0:1], c32[1:2], c32[2:3]
        self.decision_slot = tail[2: 2 + DECISION_BYTES // 8]
        self.pair_slots = tail[18: 18 + 8]
        self.offsets, self.rank, self.err = [int(o) for o in offsets], int(rank), err_flag
        self.epochs = torch.zeros(4, dtype=torch.int32, device=tail.device)    # barrier, bcast, gather (private, on the device)
        self.tp_size = len(self.offsets)
        if self.tp_size > 8:
            raise DimensionError("at most 8 ranks")

    def barrier(self) -> None:
        from .adapters import peer_barrier
        peer_barrier(self.barrier_counter, self.epochs[0:1], self.offsets, self.err)

    def broadcast_decision(self, buf: torch.Tensor) -> None:
        from .adapters import peer_bcast
        peer_bcast(buf, self.decision_slot, buf, self.rank == 0, self.bcast_counter, self.epochs[1:2], self.offsets, self.err)

    def argmax_pairs(self, val: torch.Tensor, idx: torch.Tensor, out_idx: torch.Tensor) -> None:
        from .adapters import peer_argmax
        peer_argmax(val, idx, self.pair_slots, self.rank, self.gather_counter, self.epochs[2:3], self.offsets, out_idx, self.err)

    def all_reduce_sum(self, t: torch.Tensor) -> None:   # pragma: no cover - the push step has no separate all-reduce
        raise StateError("tp_push: the sums are pushed from the GEMV epilogues")


class LlamaEngine:
    """Resident weights, expert bank, descriptor table, KV cache and the captured decode step."""

    def __init__(self, cfg: LlamaConfig, init: str = "host", device=None, group=None, comm=None, peers=None):
        cfg.validate()
        torch_ = _capi.require_cuda()
        self.cfg = cfg
        self.dev = torch_.device(device) if device is not None else torch_.device("cuda", torch_.cuda.current_device())
        if self.dev.index is None:
            self.dev = torch_.device("cuda", torch_.cuda.current_device())
        if self.dev.index != torch_.cuda.current_device():
            with torch_.cuda.device(self.dev):      # build (and configure the kernels) on the engine's own device
                self.__init__(cfg, init=init, device=self.dev, group=group, comm=comm, peers=peers)
            return
        # `comm` lets a caller supply the exchange layer (tests build one shard with no peers)
        self.comm = comm if comm is not None else Collectives(group, cfg.tp_size)
        self.step_comm = self.comm          # what the decode step calls; a tp_push engine swaps in PeerCollectives
        self.recorder = DispatchRecorder()
        d, hd = cfg.hidden, cfg.head_dim
        shp = cfg.segment_shapes()
        self.q_rows, self.kv_rows, self.ffn_local = shp["q"][0], shp["k"][0], shp["gate"][0]
        self.heads_local, self.kv_local = self.q_rows // hd, self.kv_rows // hd
        self.vocab_local = cfg.vocab // cfg.tp_size
        bf = torch.bfloat16
        dev = self.dev
        if init not in ("host", "device"):
            raise ValueError("init must be 'host' (PCG64, reproducible on the CPU oracle) or 'device' (throughput runs)")
        gen = torch.Generator(device=dev)
        gen.manual_seed(cfg.seed * 1000003 + cfg.tp_rank)

        def dev_uniform(shape, fan_in, dtype=bf):
            t = torch.empty(shape, dtype=torch.float32, device=dev).uniform_(-1.0, 1.0, generator=gen)
            return t.mul_(fan_in ** -0.5).to(dtype)

        hw = host_weights(cfg) if init == "host" else None

        def put(a, dtype=bf):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype).contiguous()

        self.embed = Matrix(put(hw["embed"]) if hw else dev_uniform((cfg.vocab, d), d), "bf16")
        self.router = Matrix(put(hw["router"]) if hw else dev_uniform((cfg.experts, d), d), "bf16")
        self.lm_head = Matrix(put(hw["lm_head"]) if hw else dev_uniform((self.vocab_local, d), d), "bf16")
        self.final_norm = put(hw["final_norm"], torch.float32) if hw else torch.ones(d, dtype=torch.float32, device=dev)
        self.wqkv, self.wo, self.wgu, self.wdown = [], [], [], []
        self.attn_norm, self.ffn_norm = [], []
        targets, downs, ups = [], [], []
        for li in range(cfg.layers):
            qkv = torch.empty((self.q_rows + 2 * self.kv_rows, d), dtype=bf, device=dev)
            gu = torch.empty((2 * self.ffn_local, d), dtype=bf, device=dev)
            wo = torch.empty((d, self.q_rows), dtype=bf, device=dev)
            wdn = torch.empty((d, self.ffn_local), dtype=bf, device=dev)
            views = {
                "q": qkv[: self.q_rows], "k": qkv[self.q_rows: self.q_rows + self.kv_rows], "v": qkv[self.q_rows + self.kv_rows:],
                "o": wo, "gate": gu[: self.ffn_local], "up": gu[self.ffn_local:], "down": wdn,
            }
            for name in SEGMENT_NAMES:
                d_out, d_in = shp[name]
                if hw:
                    views[name].copy_(put(hw["layers"][li][name]["w"]))
                    dn, up = put(hw["layers"][li][name]["down"]), put(hw["layers"][li][name]["up"])
                else:
                    views[name].copy_(dev_uniform((d_out, d_in), cfg.full_segment_shapes()[name][1]))
                    dn = dev_uniform((cfg.experts, cfg.rank, d_in), cfg.full_segment_shapes()[name][1])
                    up = dev_uniform((cfg.experts, d_out, cfg.rank), cfg.rank)
                targets.append(Matrix(views[name], "bf16"))
                downs.append(dn)
                ups.append(up)
            self.wqkv.append(qkv)
            self.wo.append(wo)
            self.wgu.append(gu)
            self.wdown.append(wdn)
            self.attn_norm.append(put(hw["layers"][li]["attn_norm"], torch.float32) if hw else torch.ones(d, dtype=torch.float32, device=dev))
            self.ffn_norm.append(put(hw["layers"][li]["ffn_norm"], torch.float32) if hw else torch.ones(d, dtype=torch.float32, device=dev))
        self.targets, self.bank_down, self.bank_up = targets, downs, ups
        self.pristine = [t.copy() for t in targets] if (cfg.adapters and cfg.keep_pristine) else None
        self.table = SwitchTable(targets, downs, ups, pristine=self.pristine) if cfg.adapters else None
        # stacked ranks one launch takes: 256 on the tcgen05 path (K-chunked), 64 otherwise; beyond it the switch
        # runs as several tensor-path passes (rank-64 tables, tables off the tcgen05 path)
        self.rank_limit = self.table.one_launch_ranks() if self.table is not None else 0
        self.split_switch = bool(self.table is not None and cfg.split_switch and self.table.info()["tensor_path"]
                                 and cfg.rank <= self.rank_limit)
        cos, sin = rope_tables(cfg)
        self.cos, self.sin = put(cos, torch.float32), put(sin, torch.float32)
        self.k_cache = [torch.zeros((self.kv_local, cfg.max_seq, hd), dtype=bf, device=dev) for _ in range(cfg.layers)]
        self.v_cache = [torch.zeros((self.kv_local, cfg.max_seq, hd), dtype=bf, device=dev) for _ in range(cfg.layers)]
        # per-step device state
        f32 = torch.float32
        self.x = [torch.zeros(d, dtype=f32, device=dev) for _ in range(2)]
        self.qkv_buf = torch.zeros(self.q_rows + 2 * self.kv_rows, dtype=f32, device=dev)
        self.attn_buf = torch.zeros(self.q_rows, dtype=f32, device=dev)
        self.gu_buf = torch.zeros(2 * self.ffn_local, dtype=f32, device=dev)
        self.logits = torch.zeros(self.vocab_local, dtype=f32, device=dev)
        self.token_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        # what a step reports back: [next token, status word].  Every kernel of the engine that validates on the device
        # (unusable decision, phase-barrier timeout) raises into report[1]; decode_step reads both words in ONE copy.
        self.report = torch.zeros(2, dtype=torch.int32, device=dev)
        self.next_dev, self.err_dev = self.report[0:1], self.report[1:2]
        self._pin_in = torch.zeros(1, dtype=torch.int32).pin_memory()
        self._pin_out = torch.zeros(2, dtype=torch.int32).pin_memory()
        self._pin_in_np, self._pin_out_np = self._pin_in.numpy(), self._pin_out.numpy()
        self._done_evt = torch.cuda.Event()
        # host mirrors of the device counters (the device advances them itself, af_step_advance; the host only needs
        # them to refuse a step past the KV cache and to pick the refreshing launch -- no read-back)
        self._pos_host = 0
        self._steps_host = 0
        self.auto_graph = True      # decode_step replays the captured step (see decode_step)
        self.refresh_every = cfg.refresh_every if (cfg.adapters and cfg.keep_pristine and cfg.switch_mode == "inplace") else 0
        if self.table is not None:
            _capi.check(_capi.lib().af_table_set_error_word(self.table.device_table.handle, _ptr(self.err_dev)))
        self.next_val = torch.zeros(1, dtype=f32, device=dev)
        self.pos_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.cur = DeviceDecision(dev)
        self.prev = DeviceDecision(dev)
        self.have_prev = False
        self.history = torch.zeros(cfg.max_seq, dtype=torch.int32, device=dev)
        sm_count = _capi.device_info()["sm_count"]
        # grid of the decode attention: sized for the longest context (one split per 32 positions, at most 8 --
        # measured: 1 split costs 13 % of the step at 400 positions, 12 or 16 cost more than 8 even at 1800);
        # the kernel itself uses fewer splits while the context is short
        if cfg.attn_splits > 0:
            self.attn_splits = cfg.attn_splits
        elif hd in (64, 128):    # attn_decode2_kernel: 64-position splits staged in shared memory, up to 32 per head
            self.attn_splits = max(1, min(32, -(-cfg.max_seq // 64)))
        else:
            self.attn_splits = 1 if cfg.max_seq <= 64 else min(8, -(-cfg.max_seq // 32))
        self.attn_ws = torch.zeros(self.heads_local * self.attn_splits * (hd + 2), dtype=f32, device=dev)
        self.attn_tickets = torch.zeros(self.heads_local, dtype=torch.int32, device=dev)
        self.forced_dev = None
        self._graphs = {}
        # phase counters of the chained plain-GEMV launches (4 per layer), zeroed once per forward
        self.use_gemv_chain = cfg.gemv_chain and cfg.tp_size == 1
        self.gc_done = torch.zeros(4 * cfg.layers, dtype=torch.int32, device=dev)
        # the whole plain forward as one launch over a device-side phase table (head_dim 64 / 128, single rank)
        self.use_fw_persistent = bool(self.use_gemv_chain and cfg.persistent_forward and hd in (64, 128)
                                      and os.environ.get("AF_FW_PERSISTENT", "1") != "0")
        self._fw = None
        if self.use_fw_persistent:
            self._fw_build()            # (uploads the phase table: not something to do lazily inside a graph capture)
        # ---- fused switch + GEMV ("chase") ----
        want = cfg.forward_mode
        # more stacked ranks than one launch takes: the switch runs in tensor-path passes and the LAST pass carries the GEMVs
        steady_ranks = (1 if cfg.switch_mode == "from_pristine" else 2) * cfg.top_k * cfg.rank
        self.chase_split = bool(self.split_switch and steady_ranks > self.rank_limit)
        can = cfg.adapters and self.table is not None and self.table.info()["tensor_path"] \
            and (steady_ranks <= self.rank_limit or self.chase_split) and cfg.compute in ("auto", "mma")
        if want == "chase" and not can:
            raise ConfigError("forward_mode='chase' needs the tensor path (bf16, rank % 8 == 0) and a steady switch of at most "
                              f"{self.rank_limit} stacked ranks in one launch")
        self.chase = can and want in ("auto", "chase")
        if self.chase:
            # launches of one token: [qkv(0)] attn [o gu down qkv(1)] attn ... [o gu down (L-1)]
            # TP: the row-parallel projections (o, down) end in an all-reduce of their fixed-point accumulators
            # (exact: integer sums), so the phases cannot share one launch -- one launch per projection
            # ... unless the epilogue does the all-reduce itself (tp_push): o and down add their partial sums into EVERY
            # rank's accumulators over peer memory and the phase counters count the CTAs of all ranks -- the single-rank
            # chain, unchanged, is then the TP step
            n_qkv, n_gu = self.q_rows + 2 * self.kv_rows, 2 * self.ffn_local
            per_layer = n_qkv + d + n_gu + d
            arena_words = cfg.layers * (per_layer + 2)
            self.tp_push, self.peer_buf = False, None
            env_push = os.environ.get("AF_TP_PUSH", "1") != "0"
            if cfg.tp_push is not None:
                want_push = cfg.tp_push
            else:   # automatic: a real process group whose ranks are this engine's TP ranks (or a caller-supplied buffer)
                import torch.distributed as dist
                have_group = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) == cfg.tp_size
                want_push = cfg.tp_size > 1 and env_push and (peers is not None or have_group)
            push_ok = cfg.chain and bool(self.table.info().get("umma_path")) and not self.chase_split
            if cfg.tp_push and not push_ok:
                raise ConfigError("tp_push needs the chained launches on the tcgen05 path (chain=True, umma_path, one-launch switch)")
            if want_push and push_ok:
                try:
                    # (+ a tail behind the arena that is never zeroed: the counters of the barrier / broadcast / argmax, their slots)
                    n_buf = arena_words + PEER_TAIL_WORDS
                    if peers is not None:
                        self.peer_buf = peers(n_buf)
                    elif cfg.tp_size == 1:
                        self.peer_buf = PeerBuffer.local(n_buf, dev)
                    else:
                        self.peer_buf = PeerBuffer.symmetric(n_buf, dev, group)
                    # (a one-entry list on a TP shard: the shard runs ALONE -- scripts/bench_shard.py times a rank's step that way)
                    if len(self.peer_buf.offsets) not in (1, cfg.tp_size) or self.peer_buf.tensor.numel() < arena_words + PEER_TAIL_WORDS:
                        raise ConfigError(f"the peer buffer maps {len(self.peer_buf.offsets)} rank(s) for tp_size {cfg.tp_size}, "
                                          "or is smaller than the arena")
                    self.tp_push = True
                except (RuntimeError, ImportError, AttributeError, TypeError, ConfigError) as e:   # no peer access between the ranks:
                    if cfg.tp_push:                                                       # NCCL all-reduces instead
                        raise
                    self.peer_buf = None
                    self.tp_push_unavailable = f"{type(e).__name__}: {e}"
            self.chase_chained = cfg.chain and (cfg.tp_size == 1 or self.tp_push)
            seg = lambda li: {"qkv": [7 * li, 7 * li + 1, 7 * li + 2], "o": [7 * li + 3], "gu": [7 * li + 4, 7 * li + 5],  # noqa: E731
                              "down": [7 * li + 6]}                                 # SEGMENT_NAMES order: q k v o gate up down
            self.groups = []
            for li in range(cfg.layers):
                sg = seg(li)
                if self.chase_chained:
                    mid = [sg["o"], sg["gu"], sg["down"]] + ([seg(li + 1)["qkv"]] if li + 1 < cfg.layers else [])
                    self.groups.append({"qkv": SegmentGroup(self.table, sg["qkv"]) if li == 0 else None,
                                        "mid": SegmentGroup(self.table, mid)})
                    if self.tp_push:            # phases 0 (o) and 2 (down) are row-parallel
                        self.groups[-1]["mid"].set_peers(self.peer_buf.offsets, reduce_phases=[0, 2])
                elif cfg.chain:
                    # TP: the chain breaks only where a collective sits -- after o and after down.  gate|up -> down has
                    # none in between (column-parallel outputs feed the row-parallel input shard locally): one launch.
                    self.groups.append({"qkv": SegmentGroup(self.table, sg["qkv"]), "o": SegmentGroup(self.table, sg["o"]),
                                        "gudown": SegmentGroup(self.table, [sg["gu"], sg["down"]])})
                else:
                    self.groups.append({k: SegmentGroup(self.table, v) for k, v in sg.items()})
            # fixed-point accumulators of every launch of a token and the chains' phase counters:
            # one arena, zeroed once per step
            if self.tp_push:
                self.acc_arena = self.peer_buf.tensor[:arena_words]
                self.peer_comm = PeerCollectives(self.peer_buf.tensor[arena_words: arena_words + PEER_TAIL_WORDS], self.peer_buf.offsets,
                                                 cfg.tp_rank if len(self.peer_buf.offsets) > 1 else 0, self.err_dev)
                self.peer_counter, self.peer_epoch = self.peer_comm.barrier_counter, self.peer_comm.epochs[0:1]
                # the engine's own exchange layer is replaced too (a caller-supplied `comm` -- tests, a shard timed alone -- stays)
                if comm is None:
                    self.step_comm = self.peer_comm
            else:
                self.acc_arena = torch.zeros(arena_words, dtype=torch.int64, device=dev)
            self.acc = []
            self.phase_done = []
            # tcgen05 path: RMSNorm scales are deferred -- one CTA computes them, the consumers of q|k|v
            # (attention) and gate|up (the SiLU prologue of the down projection) apply them
            stacked = (1 if cfg.switch_mode == "from_pristine" else 2) * cfg.top_k * cfg.rank   # ranks of a steady switch
            # af_api.cu: stacked ranks the tcgen05 chain kernel takes
            umma_ranks = min(int(os.environ.get("AF_UMMA_MAX_RANKS_CHAIN", "256")), self.rank_limit)
            self.defer_norm = bool(self.table.info().get("umma_path")) and cfg.defer_norm and stacked <= umma_ranks
            self.inv_qkv = torch.ones(cfg.layers, dtype=torch.float32, device=dev)
            self.inv_gu = torch.ones(cfg.layers, dtype=torch.float32, device=dev)
            counters = self.acc_arena[cfg.layers * per_layer:].view(torch.int32)   # 4 int32 per layer
            for li in range(cfg.layers):
                o = li * per_layer
                self.acc.append({"qkv": self.acc_arena[o: o + n_qkv], "o": self.acc_arena[o + n_qkv: o + n_qkv + d],
                                 "gu": self.acc_arena[o + n_qkv + d: o + n_qkv + d + n_gu],
                                 "down": self.acc_arena[o + n_qkv + d + n_gu: o + per_layer]})
                self.phase_done.append(counters[4 * li: 4 * li + 4])
            self.schedule_shares = None
            if cfg.calibrate and self.chase_chained and self.pristine is not None and cfg.layers >= 4 \
                    and os.environ.get("AF_CALIBRATE", "1") != "0":
                self.calibrate_schedule()

    # -- the pieces of one step ---------------------------------------------------------

    def _check(self, status):
        _capi.check(status)

    def pregate(self) -> DeviceDecision:
        """Pre-gate on the embedding row of *token_dev (model.py:342-343), then broadcast."""
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        if cfg.tp_rank == 0 or cfg.tp_size == 1:
            self._check(L.af_pregate(_ptr(self.router.data), _capi.AF_BF16, cfg.experts, cfg.hidden, _ptr(self.embed.data),
                                     _capi.AF_BF16, _ptr(self.token_dev), cfg.top_k, self.cur.ptr, None, st))
        self.step_comm.broadcast_decision(self.cur.buf)
        return self.cur

    @_on_device
    def fused_switch(self, prev, cur, **kw) -> None:
        """W <- W + delta(cur) - delta(prev) over all 7 x L local shards, one launch."""
        if self.table is None:
            raise StateError("this engine was built without adapters")
        kw.setdefault("max_k", self.cfg.top_k)
        kw.setdefault("compute", self.cfg.compute)
        cfg = self.cfg
        blocks = (cfg.top_k if (prev is not None and kw.get("mode", "inplace") == "inplace") else 0) + (cfg.top_k if cur is not None else 0)
        if self.split_switch and blocks * cfg.rank > self.rank_limit and kw["compute"] in ("auto", "mma") \
                and all(isinstance(dec, DeviceDecision) for dec in (prev, cur) if dec is not None):
            # more stacked ranks than one tensor-path launch holds (Llama-2-70B): a few tensor-path passes
            # instead of one FMA-bound CUDA-core pass
            self.table.switch_in_passes(prev, cur, rank=cfg.rank, max_k=cfg.top_k, mode=kw.get("mode", "inplace"),
                                        compute=kw["compute"], scale=kw.get("scale", 1.0))
            return
        self.table.switch(prev, cur, **kw)

    def merge(self, dec, **kw) -> None:
        self.fused_switch(None, dec, **kw)

    def unmerge(self, dec, **kw) -> None:
        self.fused_switch(dec, None, **kw)

    def _switch_for_step(self, with_prev: bool, refresh: bool = False) -> None:
        if self.cfg.switch_mode == "from_pristine" or refresh:
            self.fused_switch(None, self.cur, mode="from_pristine")   # refresh: model.py:344-349 + the merge, in one pass
        else:
            self.fused_switch(self.prev if with_prev else None, self.cur)

    def calibrate_schedule(self, rounds: int = 2) -> None:
        """Measure how long every CTA of the chained launches spends in each phase (the library's timeline probe,
        `af_set_timeline`) and rebuild the launches' schedules with the phases' tiles split by the measured rates
        (`af_chain_create_weighted`).  A launch's CTAs meet at every phase barrier, so the slowest SM sets the pace of
        the phase; the rates differ by a few per cent with an SM's position and are the same in every launch.  Changes
        which CTA takes which tile and nothing else (weights and accumulators bit-identical).  Runs a few decode steps
        on a scratch token stream and restores the engine (pristine weights, position 0) afterwards."""
        cfg, L = self.cfg, _capi.lib()
        if not (self.chase and self.chase_chained and self.pristine is not None):
            raise StateError("schedule calibration applies to the chained one-pass schedule with a pristine copy")
        grid = _capi.device_info()["sm_count"]
        slots = _capi.AF_TIMELINE_SLOTS
        n_launch = cfg.layers + 1
        shares = np.ones((4, grid), dtype=np.float64)
        scratch = np.random.Generator(np.random.PCG64(12345)).integers(0, cfg.vocab, 16)
        for _ in range(rounds):
            self.reset(forced=scratch)
            for _ in range(2):
                self.decode_step(graph=False)
            buf = torch.zeros(n_launch * grid * slots, dtype=torch.int64, device=self.dev)
            self._check(L.af_set_timeline(_ptr(buf), n_launch, grid * slots))
            try:
                self.decode_step(graph=False)
            finally:
                self._check(L.af_set_timeline(None, 0, 0))
            tl = buf.cpu().numpy().reshape(n_launch, grid, slots).astype(np.float64)
            tl[tl == 0] = np.nan
            mid = tl[2:cfg.layers - 1]                                    # the four-phase launches of the inner layers
            new = shares.copy()
            for ph in range(1, 4):                                        # (phase 0, o, is a handful of tiles: start skew, not rate)
                start = mid[:, :, 9 + 4 * ph]                             # barrier passed
                end = mid[:, :, 8 + 4 * (ph + 1)] if ph < 3 else mid[:, :, 7]   # next phase's wait begins / consumers done
                dur = np.nanmean(end - start, axis=0)                     # [cta]
                if not np.all(np.isfinite(dur)) or np.nanmin(dur) <= 0:
                    continue
                rel = np.nanmedian(dur) / dur                             # > 1: this CTA was early and can take more
                new[ph] = shares[ph] * (1.0 + 0.8 * (np.clip(rel, 0.8, 1.25) - 1.0))
            shares = new / new.mean(axis=1, keepdims=True)
            self._rebuild_mid_groups(shares)
        self.schedule_shares = shares
        self.reset()

    def _rebuild_mid_groups(self, shares) -> None:
        cfg = self.cfg
        seg = lambda li: {"qkv": [7 * li, 7 * li + 1, 7 * li + 2], "o": [7 * li + 3], "gu": [7 * li + 4, 7 * li + 5], "down": [7 * li + 6]}  # noqa: E731
        for li in range(cfg.layers):
            sg = seg(li)
            mid = [sg["o"], sg["gu"], sg["down"]] + ([seg(li + 1)["qkv"]] if li + 1 < cfg.layers else [])
            old = self.groups[li]["mid"]
            self.groups[li]["mid"] = SegmentGroup(self.table, mid, cta_share=[list(shares[ph]) for ph in range(len(mid))])
            old.close()
        self._graphs = {}

    def _gv_phase(self, w, rows, cols, x, out, prologue=0, norm_w=None, eps=0.0, epilogue=0, res=None):
        return _capi.GvPhase(w=_ptr(w), rows=rows, cols=cols, ld=cols, x=_ptr(x), out=_ptr(out), res=_ptr(res) if res is not None else None,
                             norm_w=_ptr(norm_w) if norm_w is not None else None, eps=float(eps), prologue=prologue, epilogue=epilogue)

    def forward_chained(self) -> None:
        """The same forward as `forward`, with o -> gate|up -> down -> next q|k|v (-> lm_head for
        the last layer) as ONE persistent launch per layer (af_gemv_chain): the weights of the four
        projections stream back to back while the consumers hop over the phase boundaries."""
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        d, eps = cfg.hidden, cfg.rms_eps
        xa, xb = self.x
        n_qkv, n_gu = self.q_rows + 2 * self.kv_rows, 2 * self.ffn_local
        self.gc_done.zero_()
        self._check(L.af_embed(_ptr(self.embed.data), _capi.AF_BF16, d, _ptr(self.token_dev), _ptr(xa), st))
        self._check(L.af_gemv_fused(_ptr(self.wqkv[0]), n_qkv, d, d, _ptr(xa), _ptr(self.qkv_buf), _capi.AF_PRO_RMSNORM,
                                    _ptr(self.attn_norm[0]), eps, _capi.AF_EPI_NONE, None, st))
        for li in range(cfg.layers):
            self._check(L.af_attn_decode(_ptr(self.qkv_buf), _ptr(self.k_cache[li]), _ptr(self.v_cache[li]), _ptr(self.cos),
                                         _ptr(self.sin), _ptr(self.pos_dev), self.heads_local, self.kv_local, cfg.head_dim,
                                         cfg.max_seq, self.attn_splits, _ptr(self.attn_ws), _ptr(self.attn_tickets),
                                         _ptr(self.attn_buf), st))
            phases = [
                self._gv_phase(self.wo[li], d, self.q_rows, self.attn_buf, xb, epilogue=_capi.AF_EPI_RESIDUAL, res=xa),
                self._gv_phase(self.wgu[li], n_gu, d, xb, self.gu_buf, prologue=_capi.AF_PRO_RMSNORM, norm_w=self.ffn_norm[li], eps=eps),
                self._gv_phase(self.wdown[li], d, self.ffn_local, self.gu_buf, xa, prologue=_capi.AF_PRO_SILU_MUL,
                               epilogue=_capi.AF_EPI_RESIDUAL, res=xb),
            ]
            if li + 1 < cfg.layers:
                phases.append(self._gv_phase(self.wqkv[li + 1], n_qkv, d, xa, self.qkv_buf, prologue=_capi.AF_PRO_RMSNORM,
                                             norm_w=self.attn_norm[li + 1], eps=eps))
            else:
                phases.append(self._gv_phase(self.lm_head.data, self.vocab_local, d, xa, self.logits, prologue=_capi.AF_PRO_RMSNORM,
                                             norm_w=self.final_norm, eps=eps))
            arr = (_capi.GvPhase * len(phases))(*phases)
            self._check(L.af_gemv_chain(arr, len(phases), _ptr(self.gc_done[4 * li: 4 * li + 4]), _ptr(self.err_dev), 1, st))
        self._check(L.af_argmax_val(_ptr(self.logits), self.vocab_local, 0, _ptr(self.next_dev), _ptr(self.next_val), st))

    def _fw_build(self):
        """The device-side phase table of `forward_persistent`: q|k|v(0), then per layer attention partials, attention
        combine, o, gate|up, down and the next layer's q|k|v (the lm_head after the last layer)."""
        import ctypes

        cfg, L = self.cfg, _capi.lib()
        d, eps = cfg.hidden, cfg.rms_eps
        xa, xb = self.x
        n_qkv, n_gu = self.q_rows + 2 * self.kv_rows, 2 * self.ffn_local
        P = _capi.FwPhase

        def gemv(w, rows, cols, x, out, prologue=_capi.AF_PRO_NONE, norm_w=None, epilogue=_capi.AF_EPI_NONE, res=None):
            return P(w=_ptr(w), x=_ptr(x), out=_ptr(out), res=_ptr(res) if res is not None else None,
                     norm_w=_ptr(norm_w) if norm_w is not None else None, k_cache=None, v_cache=None, ld=cols, rows=rows, cols=cols,
                     eps=float(eps), prologue=prologue, epilogue=epilogue, kind=_capi.AF_FW_GEMV)

        ph = [gemv(self.wqkv[0], n_qkv, d, xa, self.qkv_buf, _capi.AF_PRO_RMSNORM, self.attn_norm[0])]
        for li in range(cfg.layers):
            ph.append(P(w=None, x=_ptr(self.qkv_buf), out=None, res=None, norm_w=None, k_cache=_ptr(self.k_cache[li]),
                        v_cache=_ptr(self.v_cache[li]), ld=0, rows=0, cols=0, eps=0.0, prologue=0, epilogue=0, kind=_capi.AF_FW_ATTN_PARTIAL))
            ph.append(P(w=None, x=None, out=_ptr(self.attn_buf), res=None, norm_w=None, k_cache=None, v_cache=None, ld=0, rows=0, cols=0,
                        eps=0.0, prologue=0, epilogue=0, kind=_capi.AF_FW_ATTN_COMBINE))
            ph.append(gemv(self.wo[li], d, self.q_rows, self.attn_buf, xb, epilogue=_capi.AF_EPI_RESIDUAL, res=xa))
            ph.append(gemv(self.wgu[li], n_gu, d, xb, self.gu_buf, _capi.AF_PRO_RMSNORM, self.ffn_norm[li]))
            ph.append(gemv(self.wdown[li], d, self.ffn_local, self.gu_buf, xa, _capi.AF_PRO_SILU_MUL, epilogue=_capi.AF_EPI_RESIDUAL, res=xb))
            if li + 1 < cfg.layers:
                ph.append(gemv(self.wqkv[li + 1], n_qkv, d, xa, self.qkv_buf, _capi.AF_PRO_RMSNORM, self.attn_norm[li + 1]))
            else:
                ph.append(gemv(self.lm_head.data, self.vocab_local, d, xa, self.logits, _capi.AF_PRO_RMSNORM, self.final_norm))
        arr = (P * len(ph))(*ph)
        max_cols = ctypes.c_int32()
        self._check(L.af_forward_validate(arr, len(ph), self.heads_local, self.kv_local, cfg.head_dim, ctypes.byref(max_cols)))
        raw = np.frombuffer(ctypes.string_at(ctypes.addressof(arr), ctypes.sizeof(arr)), dtype=np.uint8).copy()
        chunks = -(-cfg.max_seq // 64)
        self._fw = {"table": torch.from_numpy(raw).to(self.dev), "n": len(ph), "max_cols": int(max_cols.value),
                    "done": torch.zeros(len(ph), dtype=torch.int32, device=self.dev),
                    "ws": torch.zeros(self.heads_local * chunks * (cfg.head_dim + 2), dtype=torch.float32, device=self.dev)}

    def forward_persistent(self) -> None:
        """The same forward as `forward`, as ONE persistent launch over all layers (af_forward_persistent): the CTAs
        never leave between projections and attentions; the weights of the next projection fill the ring while the
        attention of the layer runs as two phases of the same kernel."""
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        if self._fw is None:
            self._fw_build()
        fw = self._fw
        fw["done"].zero_()
        self._check(L.af_embed(_ptr(self.embed.data), _capi.AF_BF16, cfg.hidden, _ptr(self.token_dev), _ptr(self.x[0]), st))
        self._check(L.af_forward_persistent(_ptr(fw["table"]), fw["n"], fw["max_cols"], _ptr(self.cos), _ptr(self.sin), _ptr(self.pos_dev),
                                            self.heads_local, self.kv_local, cfg.head_dim, cfg.max_seq, _ptr(fw["ws"]), _ptr(fw["done"]),
                                            _ptr(self.err_dev), 1, st))
        self._check(L.af_argmax_val(_ptr(self.logits), self.vocab_local, 0, _ptr(self.next_dev), _ptr(self.next_val), st))

    def forward(self) -> None:
        """Merged-path forward of one token (model.py:367-371 on the Llama block)."""
        if self.use_fw_persistent:
            return self.forward_persistent()
        if self.use_gemv_chain:
            return self.forward_chained()
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        d, eps = cfg.hidden, cfg.rms_eps
        tp = cfg.tp_size
        res_epi = _capi.AF_EPI_RESIDUAL if (tp == 1 or cfg.tp_rank == 0) else _capi.AF_EPI_NONE
        xa, xb = self.x
        self._check(L.af_embed(_ptr(self.embed.data), _capi.AF_BF16, d, _ptr(self.token_dev), _ptr(xa), st))
        for li in range(cfg.layers):
            self._check(L.af_gemv_fused(_ptr(self.wqkv[li]), self.q_rows + 2 * self.kv_rows, d, d, _ptr(xa), _ptr(self.qkv_buf),
                                        _capi.AF_PRO_RMSNORM, _ptr(self.attn_norm[li]), eps, _capi.AF_EPI_NONE, None, st))
            self._check(L.af_attn_decode(_ptr(self.qkv_buf), _ptr(self.k_cache[li]), _ptr(self.v_cache[li]), _ptr(self.cos),
                                         _ptr(self.sin), _ptr(self.pos_dev), self.heads_local, self.kv_local, cfg.head_dim,
                                         cfg.max_seq, self.attn_splits, _ptr(self.attn_ws), _ptr(self.attn_tickets),
                                         _ptr(self.attn_buf), st))
            self._check(L.af_gemv_fused(_ptr(self.wo[li]), d, self.q_rows, self.q_rows, _ptr(self.attn_buf), _ptr(xb),
                                        _capi.AF_PRO_NONE, None, 0.0, res_epi, _ptr(xa) if res_epi else None, st))
            self.comm.all_reduce_sum(xb)
            self._check(L.af_gemv_fused(_ptr(self.wgu[li]), 2 * self.ffn_local, d, d, _ptr(xb), _ptr(self.gu_buf),
                                        _capi.AF_PRO_RMSNORM, _ptr(self.ffn_norm[li]), eps, _capi.AF_EPI_NONE, None, st))
            self._check(L.af_gemv_fused(_ptr(self.wdown[li]), d, self.ffn_local, self.ffn_local, _ptr(self.gu_buf), _ptr(xa),
                                        _capi.AF_PRO_SILU_MUL, None, 0.0, res_epi, _ptr(xb) if res_epi else None, st))
            self.comm.all_reduce_sum(xa)
        self._check(L.af_gemv_fused(_ptr(self.lm_head.data), self.vocab_local, d, d, _ptr(xa), _ptr(self.logits),
                                    _capi.AF_PRO_RMSNORM, _ptr(self.final_norm), eps, _capi.AF_EPI_NONE, None, st))
        self._check(L.af_argmax_val(_ptr(self.logits), self.vocab_local, cfg.tp_rank * self.vocab_local, _ptr(self.next_dev),
                                    _ptr(self.next_val), st))
        self.step_comm.argmax_pairs(self.next_val, self.next_dev, self.next_dev)

    def forward_chase(self, with_prev: bool, refresh: bool = False) -> None:
        """Switch AND merged forward of one token in one pass over the weights: each projection's
        launch merges the selected experts into its tiles (adapters.py:236-258), multiplies the
        rounded tiles with the projection's input (model.py:288) and writes them back.  4 weight
        launches + attention per layer; RMSNorm, SiLU*up and the residual adds ride in the
        prologue of the consuming launch."""
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        d, eps = cfg.hidden, cfg.rms_eps
        xa, xb = self.x
        step_mode = "from_pristine" if refresh else cfg.switch_mode   # a refreshing token rebuilds W from W0 (model.py:344-349)
        prev = self.prev if (with_prev and step_mode == "inplace") else None
        cur, max_k, mode = self.cur, cfg.top_k, step_mode
        if self.chase_split:
            # all passes but the last as plain switch launches; the last merge pass is the one fused with the forward
            cur, max_k, mode = self.table.switch_in_passes(prev, self.cur, rank=cfg.rank, max_k=cfg.top_k, mode=step_mode,
                                                           compute=cfg.compute, hold_last=True)
            prev = None
        kw = dict(max_k=max_k, mode=mode, plan_prebuilt=True)
        self.table.build_plan(prev, cur, max_k=max_k, mode=mode)
        self.acc_arena.zero_()
        if self.tp_push:
            # nobody pushes into these accumulators before every rank has zeroed its own (af_peer_barrier: a monotonic
            # counter behind the arena, bumped on every rank by every rank)
            self.peer_comm.barrier()
        self._check(L.af_embed(_ptr(self.embed.data), _capi.AF_BF16, d, _ptr(self.token_dev), _ptr(xa), st))
        norm = "rmsnorm_deferred" if self.defer_norm else "rmsnorm"
        # timing experiment only (wrong results): AF_SKIP_ATTN=1 leaves the attention launches out -- how much of the step
        # the hand-over around them costs (Llama-2-7B, 1024 positions: 5.23 against 5.50 ms)
        skip_attn = os.environ.get("AF_SKIP_ATTN") == "1"
        for li in range(cfg.layers):
            g, a = self.groups[li], self.acc[li]
            last = li + 1 == cfg.layers
            iq = self.inv_qkv[li: li + 1] if self.defer_norm else None
            ig = self.inv_gu[li: li + 1] if self.defer_norm else None
            qkv_first = dict(acc_out=a["qkv"], xin=xa, prologue=norm, norm_w=self.attn_norm[li], eps=eps, inv_out=iq)
            if li == 0:
                g["qkv"].switch_gemv(prev, cur, pdl=False, **qkv_first, **kw)
            elif not self.chase_chained:
                g["qkv"].switch_gemv(prev, cur, a["qkv"], acc_in=self.acc[li - 1]["down"], res=xb, h_out=xa, prologue=norm,
                                     norm_w=self.attn_norm[li], eps=eps, inv_out=iq, pdl=True, **kw)
            if not skip_attn:
                self._check(L.af_attn_decode_fix(_ptr(a["qkv"]), _ptr(iq) if iq is not None else None, _ptr(self.k_cache[li]),
                                                 _ptr(self.v_cache[li]), _ptr(self.cos), _ptr(self.sin), _ptr(self.pos_dev),
                                                 self.heads_local, self.kv_local, cfg.head_dim, cfg.max_seq, self.attn_splits,
                                                 _ptr(self.attn_ws), _ptr(self.attn_tickets), _ptr(self.attn_buf), st))
            ph_o = dict(acc_out=a["o"], xin=self.attn_buf)
            ph_gu = dict(acc_out=a["gu"], acc_in=a["o"], res=xa, h_out=xb, prologue=norm, norm_w=self.ffn_norm[li], eps=eps, inv_out=ig)
            ph_down = dict(acc_out=a["down"], acc_in=a["gu"], prologue="silu_mul", inv_in=ig)
            if self.chase_chained:
                phases = [ph_o, ph_gu, ph_down]
                if not last:
                    phases.append(dict(acc_out=self.acc[li + 1]["qkv"], acc_in=a["down"], res=xb, h_out=xa, prologue=norm,
                                       norm_w=self.attn_norm[li + 1], eps=eps,
                                       inv_out=self.inv_qkv[li + 1: li + 2] if self.defer_norm else None))
                g["mid"].switch_gemv_chain(prev, cur, phases, self.phase_done[li], pdl=True, **kw)
            else:
                g["o"].switch_gemv(prev, cur, pdl=True, **ph_o, **kw)
                self.comm.all_reduce_sum(a["o"])          # TP: partial sums of the row-parallel o, as int64 (no-op on one rank)
                if "gudown" in g:
                    g["gudown"].switch_gemv_chain(prev, cur, [ph_gu, ph_down], self.phase_done[li], pdl=True, **kw)
                else:
                    g["gu"].switch_gemv(prev, cur, pdl=True, **ph_gu, **kw)
                    g["down"].switch_gemv(prev, cur, pdl=True, **ph_down, **kw)
                self.comm.all_reduce_sum(a["down"])
        if self.tp_push:
            # the last layer's down projection has no consumer inside its launch: wait until the CTAs of every rank
            # have reported it (counter 2 of the last chain) before reading the reduced sums
            from .adapters import peer_wait
            peer_wait(self.phase_done[-1][2:3], len(self.peer_buf.offsets) * self.groups[-1]["mid"].grid, self.err_dev)
        self._check(L.af_accum_to_f32(_ptr(self.acc[-1]["down"]), _ptr(xb), _ptr(xa), d, st))
        self._check(L.af_gemv_fused(_ptr(self.lm_head.data), self.vocab_local, d, d, _ptr(xa), _ptr(self.logits),
                                    _capi.AF_PRO_RMSNORM, _ptr(self.final_norm), eps, _capi.AF_EPI_NONE, None, st))
        self._check(L.af_argmax_val(_ptr(self.logits), self.vocab_local, cfg.tp_rank * self.vocab_local, _ptr(self.next_dev),
                                    _ptr(self.next_val), st))
        self.step_comm.argmax_pairs(self.next_val, self.next_dev, self.next_dev)

    def _advance(self) -> None:
        L, st = _capi.lib(), _capi.stream_ptr()
        forced = self.forced_dev
        self._check(L.af_step_advance(self.prev.ptr if self.cfg.adapters else None, self.cur.ptr if self.cfg.adapters else None,
                                      _ptr(self.pos_dev), _ptr(self.step_dev), _ptr(self.token_dev), _ptr(self.next_dev),
                                      _ptr(forced) if forced is not None else None, int(forced.numel()) if forced is not None else 0,
                                      _ptr(self.history), int(self.history.numel()), st))

    def _step_body(self, with_prev: bool, refresh: bool = False) -> None:
        if self.chase:
            self.pregate()
            self.forward_chase(with_prev, refresh)
            self._advance()
            return
        if self.cfg.adapters:
            self.pregate()
            self._switch_for_step(with_prev, refresh)
        self.forward()
        self._advance()

    def _refresh_due(self) -> bool:
        """model.py:344-349: tokens_done > 0 and tokens_done % refresh_every == 0."""
        return bool(self.refresh_every) and self.have_prev and self._steps_host > 0 and self._steps_host % self.refresh_every == 0

    def _stepped(self) -> None:
        self._pos_host += 1
        self._steps_host += 1
        self.have_prev = self.cfg.adapters

    @_on_device
    def set_position(self, pos: int) -> None:
        """Move the decode position (benchmarks that re-time a step at a fixed context length)."""
        if not 0 <= int(pos) < self.cfg.max_seq:
            raise InputError(f"position {pos!r} outside the KV cache of {self.cfg.max_seq}")
        self.pos_dev.fill_(int(pos))
        self._pos_host = int(pos)

    @_on_device
    def check(self) -> None:
        """Raise what a kernel flagged since the last check (synchronises): an unusable device decision
        (IndexError / ValueError, adapters.py:199-200), a phase-barrier timeout (DeviceError)."""
        self._pin_out.copy_(self.report, non_blocking=True)
        self._done_evt.record()
        self._done_evt.synchronize()
        self._raise_flag(int(self._pin_out_np[1]))

    def _raise_flag(self, flag: int) -> None:
        if flag:
            self.err_dev.zero_()
            _capi.raise_for_flag(flag)

    # -- public stepping ---------------------------------------------------------------------

    @_on_device
    def reset(self, first_token: int = 0, forced=None) -> None:
        """Start a new sequence: position 0, weights back to pristine, optional teacher-forced
        token stream (consumed instead of the greedy feedback)."""
        if not 0 <= int(first_token) < self.cfg.vocab:
            raise InputError(f"token {first_token!r} outside vocab of {self.cfg.vocab}")
        if self.table is not None and self.have_prev:
            if self.pristine is not None:
                self.table.refresh()
            else:
                self.unmerge(self.prev)
        self.have_prev = False
        self.pos_dev.zero_()
        self.step_dev.zero_()
        self._pos_host = self._steps_host = 0
        if forced is not None:
            forced = np.asarray(forced, dtype=np.int64)
            if forced.size == 0 or forced.min() < 0 or forced.max() >= self.cfg.vocab:
                raise InputError("teacher-forced stream is empty or leaves the vocabulary")
            self.forced_dev = torch.from_numpy(forced.astype(np.int32)).to(self.dev)
            first_token = int(forced[0])
        else:
            self.forced_dev = None
        self.token_dev.fill_(int(first_token))
        self._graphs = {}

    @_on_device
    def decode_step(self, token: int | None = None, *, graph: bool | None = None) -> int:
        """One decode step through the public API: the consumed token comes from the host (4 bytes
        H2D from a pinned word), the next token and the step's status word are read back together
        (8 bytes D2H into pinned memory) -- the one synchronisation of the step.  The step itself is
        a fixed launch sequence driven by device-resident state, so from the second token on it is
        replayed as a CUDA graph (captured on first use; `graph=False` / `auto_graph = False` keep
        the eager launches, which TP engines use unless AF_TP_GRAPH=1)."""
        if token is not None:
            if not 0 <= int(token) < self.cfg.vocab:
                raise InputError(f"token {token!r} outside vocab of {self.cfg.vocab}")
            self._pin_in_np[0] = int(token)
            self.token_dev.copy_(self._pin_in, non_blocking=True)
        if self._pos_host >= self.cfg.max_seq:
            raise StateError("KV cache is full")
        refresh = self._refresh_due()
        use_graph = self.auto_graph if graph is None else bool(graph)
        steady = self.have_prev or not self.cfg.adapters or self.cfg.switch_mode == "from_pristine"
        if use_graph and steady and self.graph_ok():
            if "steady" not in self._graphs:
                self.capture()
            self._graphs["refresh" if refresh else "steady"].replay()
        else:
            self._step_body(self.have_prev and not refresh, refresh)
        self._stepped()
        self._pin_out.copy_(self.report, non_blocking=True)
        self._done_evt.record()
        self._done_evt.synchronize()
        self._raise_flag(int(self._pin_out_np[1]))
        return int(self._pin_out_np[0])

    def graph_ok(self) -> bool:
        """May the step be captured as a CUDA graph?  One rank: yes.  Tensor parallel: when the step holds no library
        collective -- the push step with the engine's own peer exchanges -- or when AF_TP_GRAPH=1 opts torch's NCCL
        collectives into the capture."""
        if self.cfg.tp_size == 1 or os.environ.get("AF_TP_GRAPH") == "1":
            return True
        return bool(getattr(self, "tp_push", False)) and self.step_comm is getattr(self, "peer_comm", None)

    @_on_device
    def capture(self) -> None:
        """Capture the steady-state step (switch with a previous decision) as a CUDA graph -- and, with
        refresh_every, the refreshing step (from-pristine switch of the current decision) as a second one."""
        if not self.have_prev and self.cfg.adapters and self.cfg.switch_mode == "inplace":
            raise StateError("run one eager decode_step first: the steady graph unmerges a previous decision")
        if not self.graph_ok():
            # torch's NCCL collectives can be captured (each rank captures its own graph after eager warm-up steps
            # have created the communicator); verified here only on a one-rank NCCL group
            # (tests/test_gpu_llama.py::test_tp_step_with_nccl_collectives_captures), hence opt-in
            raise StateError("TP steps run eagerly unless AF_TP_GRAPH=1")
        variants = [("steady", True, False)] + ([("refresh", False, True)] if self.refresh_every else [])
        for name, with_prev, refresh in variants:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    self._step_body(with_prev, refresh)
            torch.cuda.current_stream().wait_stream(side)
            self._graphs[name] = g

    @_on_device
    def replay(self) -> None:
        """One captured step, asynchronously (no read-back: `check()` / `tokens()` synchronise)."""
        if self._pos_host >= self.cfg.max_seq:
            raise StateError("KV cache is full")       # the kernels would run past the caches and the rotary tables
        self._graphs["refresh" if self._refresh_due() else "steady"].replay()
        self._stepped()

    def steps_done(self) -> int:
        return int(self.step_dev.item())

    def tokens(self, n: int | None = None) -> list:
        self.check()
        n = self.steps_done() if n is None else n
        return [int(v) for v in self.history[:n].cpu().numpy()]

    @_on_device
    def prefill(self, prompt, use_graph: bool = True) -> int:
        """Batched UNMERGED prefill of a whole prompt (model.py:408-425; PAPER Eq. 2): all T tokens go
        through every layer at once, token t with its own pre-gated decision,

            Y = X W^T + ((X A_all^T) * G) B_all^T        G[t, e*r .. e*r+r) = gate weight of expert e for token t

        i.e. three dense GEMMs per projection (grouped over the experts by stacking them), causal
        attention over the prompt, and the backbone is never written -- the reference's prefill
        never runs an sgmm either.  The GEMMs and the attention are library calls (cuBLAS bf16 with f32
        accumulation and output, the f32 activations split hi + lo; torch SDPA): this path is outside the decode metric and, as in the
        paper, not tuned; the router decisions come from the same `pregate_kernel` the decode uses.
        Fills the KV cache for positions 0 .. T-1 (bf16, rotated, as the decode kernel stores
        them), leaves the engine at position T with pristine weights, and returns the token
        emitted after the prompt.  Single rank.

        The pass is ~100 small device operations per layer and was bound by their host launches (54 of 61 ms for
        512 tokens of Llama-2-7B): with `use_graph` (default) the whole pass is captured once per prompt LENGTH as a
        CUDA graph (after one eager run that also warms the library handles) and replayed -- the prompt's tokens are
        the graph's only input."""
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise InputError("prompt must contain at least one token")
        if any(not 0 <= t < cfg.vocab for t in prompt):
            raise InputError(f"prompt leaves the vocabulary of {cfg.vocab}")
        if len(prompt) > cfg.max_seq:
            raise InputError("prompt exceeds max_seq")
        if cfg.tp_size != 1:
            raise StateError("batched prefill is single-rank; TP engines consume the prompt step by step")
        self.reset(prompt[0])
        T = len(prompt)
        if not hasattr(self, "_prefill_graphs"):
            self._prefill_graphs = {}
            self._prefill_hidden = torch.zeros(cfg.hidden, dtype=torch.float32, device=self.dev)
        host_tok = torch.tensor(prompt, dtype=torch.int32)
        entry = self._prefill_graphs.get(T) if use_graph else None
        if entry is None:
            tok = host_tok.to(self.dev)
            self._prefill_body(tok, T)                      # eager (first use of a length; also the non-graph path)
            if use_graph:
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream()
                side.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(side):
                    with torch.cuda.graph(g, stream=side):
                        self._prefill_body(tok, T)
                torch.cuda.current_stream().wait_stream(side)
                if len(self._prefill_graphs) >= 4:          # a few prompt lengths at a time (each graph owns its activations)
                    self._prefill_graphs.pop(next(iter(self._prefill_graphs)))
                self._prefill_graphs[T] = (g, tok)
        else:
            g, tok = entry
            tok.copy_(host_tok)
            g.replay()
        nxt = int(self.next_dev.item())
        self.pos_dev.fill_(T)
        self._pos_host = T
        self.step_dev.fill_(T)
        self.history[T - 1] = nxt
        self.token_dev.fill_(nxt)
        self.last_prefill_hidden = self._prefill_hidden
        return nxt

    def _prefill_body(self, tok, T: int) -> None:
        """Every device operation of `prefill` for a prompt of T tokens held in `tok` (int32, device): router decisions,
        the unmerged batched layers, the KV cache rows, the emitted token in `next_dev`.  No host synchronisation, static
        shapes: capturable as a CUDA graph per prompt length."""
        cfg, L, st = self.cfg, _capi.lib(), _capi.stream_ptr()
        d, hd, f32 = cfg.hidden, cfg.head_dim, torch.float32
        nh, nkv = self.heads_local, self.kv_local
        gates = None
        if cfg.adapters:
            decs = torch.zeros((T, DECISION_BYTES), dtype=torch.uint8, device=self.dev)
            for t in range(T):   # the decode's own router kernel, one launch per prompt token (routing.py:81-89)
                self._check(L.af_pregate(_ptr(self.router.data), _capi.AF_BF16, cfg.experts, d, _ptr(self.embed.data), _capi.AF_BF16,
                                         _ptr(tok[t: t + 1]), cfg.top_k, _ptr(decs[t]), None, st))
            ids = decs.view(torch.int32)[:, 1: 1 + cfg.top_k].long()
            wts = decs.view(f32)[:, 1 + _capi.AF_MAX_K: 1 + _capi.AF_MAX_K + cfg.top_k]
            gates = torch.zeros((T, cfg.experts), dtype=f32, device=self.dev).scatter_add_(1, ids, wts)
            gates = gates.repeat_interleave(cfg.rank, dim=1)                       # [T, N r]

        def mm(x, wt):
            """f32 [T, K] x bf16 [N, K]^T -> f32 [T, N] on the tensor cores: x = hi + lo in bf16 (residual
            2^-17, the split the fused decode launches use), f32 accumulation and f32 output."""
            hi = x.to(torch.bfloat16)
            lo = (x - hi.float()).to(torch.bfloat16)
            return torch.mm(hi, wt.t(), out_dtype=f32) + torch.mm(lo, wt.t(), out_dtype=f32)

        def linear(x, li, j, w):
            y = mm(x, w)
            if gates is not None:
                a = self.bank_down[7 * li + j].reshape(cfg.experts * cfg.rank, -1)                       # [N r, d_in]
                b = self.bank_up[7 * li + j].permute(1, 0, 2).reshape(w.shape[0], -1).contiguous()       # [d_out, N r]
                y = y + mm(mm(x, a) * gates, b)
            return y

        def rmsnorm(x, w):
            return x * torch.rsqrt(x.pow(2).mean(dim=-1, keepdim=True) + cfg.rms_eps) * w

        def rope(v):   # [T, heads, hd], rotate-half
            half = hd // 2
            c, s_ = self.cos[:T, None, :], self.sin[:T, None, :]
            a, b = v[..., :half], v[..., half:]
            return torch.cat([a * c - b * s_, b * c + a * s_], dim=-1)

        x = self.embed.data[tok.long()].float()
        for li in range(cfg.layers):
            xn = rmsnorm(x, self.attn_norm[li])
            wq, wk, wv = self.wqkv[li][: self.q_rows], self.wqkv[li][self.q_rows: self.q_rows + self.kv_rows], self.wqkv[li][self.q_rows + self.kv_rows:]
            q = rope(linear(xn, li, 0, wq).view(T, nh, hd))
            k = rope(linear(xn, li, 1, wk).view(T, nkv, hd)).to(torch.bfloat16)    # the cache holds bf16; attention reads it back
            v = linear(xn, li, 2, wv).view(T, nkv, hd).to(torch.bfloat16)
            self.k_cache[li][:, :T] = k.permute(1, 0, 2)
            self.v_cache[li][:, :T] = v.permute(1, 0, 2)
            rep = nh // nkv
            kk = k.float().permute(1, 0, 2).repeat_interleave(rep, dim=0)          # [nh, T, hd]
            vv = v.float().permute(1, 0, 2).repeat_interleave(rep, dim=0)
            att = torch.nn.functional.scaled_dot_product_attention(q.permute(1, 0, 2)[None], kk[None], vv[None], is_causal=True)[0]
            x = x + linear(att.permute(1, 0, 2).reshape(T, nh * hd), li, 3, self.wo[li])
            xn = rmsnorm(x, self.ffn_norm[li])
            g = linear(xn, li, 4, self.wgu[li][: self.ffn_local])
            u = linear(xn, li, 5, self.wgu[li][self.ffn_local:])
            x = x + linear(torch.nn.functional.silu(g) * u, li, 6, self.wdown[li])
        # the emitted token: the decode's own lm_head + argmax kernels on the last position
        self._prefill_hidden[:] = x[T - 1]
        self.x[0].copy_(x[T - 1])
        self._check(L.af_gemv_fused(_ptr(self.lm_head.data), self.vocab_local, d, d, _ptr(self.x[0]), _ptr(self.logits),
                                    _capi.AF_PRO_RMSNORM, _ptr(self.final_norm), cfg.rms_eps, _capi.AF_EPI_NONE, None, st))
        self._check(L.af_argmax_val(_ptr(self.logits), self.vocab_local, 0, _ptr(self.next_dev), _ptr(self.next_val), st))

    @_on_device
    def generate(self, prompt, n_new: int, use_graph: bool = True, prefill: str = "auto") -> list:
        """Greedy generation.  prefill="batched" (default on one rank): the whole prompt in one
        unmerged batched pass (`prefill`), as the reference prefills (model.py:408-425);
        "stepwise": the prompt token by token along the merged path (token-level pre-gating makes
        merged == unmerged, PAPER Eq. 2-4).  Then n_new tokens, the steady steps as a CUDA graph."""
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise InputError("prompt must contain at least one token")
        if n_new < 1:
            raise InputError(f"n_new must be >= 1, got {n_new}")
        if len(prompt) + n_new > self.cfg.max_seq:
            raise InputError("prompt + n_new exceeds max_seq")
        if prefill not in ("auto", "batched", "stepwise"):
            raise ValueError(f"unknown prefill mode {prefill!r}")
        if prefill == "auto":
            prefill = "batched" if self.cfg.tp_size == 1 else "stepwise"
        if prefill == "batched":
            out = [self.prefill(prompt)]
        else:
            self.reset(prompt[0])
            nxt = None
            for t in prompt:
                nxt = self.decode_step(t, graph=use_graph)
            out = [nxt]
        remaining = n_new - 1
        if remaining and not self.have_prev and self.cfg.adapters and self.cfg.switch_mode == "inplace":
            out.append(self.decode_step(graph=use_graph))     # the first merge has no previous decision: eager, then the steady graph
            remaining -= 1
        if remaining and use_graph and self.cfg.tp_size == 1:
            self.capture()
            for _ in range(remaining):
                self.replay()
            torch.cuda.synchronize()
            out = out + self.tokens()[len(prompt) + len(out) - 1:]
        else:
            for _ in range(remaining):
                out.append(self.decode_step(graph=use_graph))
        self.finalize()
        return out

    @_on_device
    def finalize(self) -> None:
        """model.py:460-474: take the last delta out again."""
        if self.table is not None and self.have_prev:
            if self.cfg.switch_mode == "from_pristine":
                self.table.refresh()
            else:
                self.unmerge(self.prev)
            self.have_prev = False

    @_on_device
    def max_backbone_deviation(self) -> float:
        if self.table is None or self.pristine is None:
            raise StateError("no pristine copy kept")
        return self.table.max_deviation()

    def decision(self) -> GateDecision:
        return self.cur.to_host()


_ = DECISION_BYTES
