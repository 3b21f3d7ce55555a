"""CPU restatement of the Llama-shaped merged-path decode step (TEST INFRASTRUCTURE ONLY).

PARITY UNPINNED for the block dataflow: the reference (`lorafuse`) has no attention, norm,
RoPE or SwiGLU, so there is no reference output to pin RMSNorm -> q/k/v ->
RoPE -> GQA attention -> o -> RMSNorm -> SwiGLU against.  What IS pinned is everything the
reference defines and this file reuses from oracle.py: the router (routing.py:49-78), the
per-segment switch arithmetic (adapters.py:188-233 + linalg.py:306-346) and the argmax rule
(model.py:396).  The block itself follows the published Llama-2/3 definition (rotate-half
RoPE, pre-norm residual stream, SiLU-gated MLP), f32 arithmetic on bf16 weights, KV cache
stored in bf16 -- the same rounding points as the CUDA path.

Only tests/ may import this module.
"""

from __future__ import annotations

import numpy as np

from . import oracle as orc

SEGMENTS = ("q", "k", "v", "o", "gate", "up", "down")


def rope_tables(head_dim: int, max_seq: int, theta: float):
    half = head_dim // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.arange(max_seq, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def rmsnorm(x, w, eps):
    x = x.astype(np.float32)
    inv = np.float32(1.0) / np.sqrt(np.float32(np.mean(x.astype(np.float64) ** 2)) + np.float32(eps))
    return (x * inv * w).astype(np.float32)


def rope(v, cos, sin):
    half = v.shape[-1] // 2
    a, b = v[..., :half], v[..., half:]
    return np.concatenate([a * cos - b * sin, b * cos + a * sin], axis=-1).astype(np.float32)


class LlamaOracle:
    """weights: dict with embed/router/lm_head (f32 carrying bf16 values), final_norm, and per
    layer attn_norm/ffn_norm plus for each segment {'bits': live bf16 bit patterns (uint16),
    'down': [N][r][d_in] bf16 bits, 'up': [N][d_out][r] bf16 bits}."""

    def __init__(self, weights, *, hidden, n_heads, n_kv_heads, top_k, rope_theta, rms_eps, max_seq):
        self.w = weights
        self.d, self.nh, self.nkv, self.k = hidden, n_heads, n_kv_heads, top_k
        self.hd = hidden // n_heads
        self.eps = rms_eps
        self.cos, self.sin = rope_tables(self.hd, max_seq, rope_theta)
        n_layers = len(weights["layers"])
        self.kc = [np.zeros((n_kv_heads, max_seq, self.hd), np.float32) for _ in range(n_layers)]
        self.vc = [np.zeros((n_kv_heads, max_seq, self.hd), np.float32) for _ in range(n_layers)]
        self.pos = 0
        self.prev = None

    def route(self, token):
        x = self.w["embed"][int(token)]                       # model.py:342-343: raw embedding row
        ids, wts, _ = orc.route(self.w["router"], x, self.k)
        return ids, wts

    def switch(self, cur, from_pristine=False, pristine=None):
        """Reference f32 switch on the upcast of every live bf16 matrix (oracle.py)."""
        for li, lw in enumerate(self.w["layers"]):
            for name in SEGMENTS:
                seg = lw[name]
                if from_pristine:
                    seg["bits"][...] = pristine[li][name]
                    orc.switch_segment_bf16(seg["bits"], seg["down"], seg["up"], None, cur)
                else:
                    orc.switch_segment_bf16(seg["bits"], seg["down"], seg["up"], self.prev, cur)
        self.prev = cur

    def forward(self, token):
        d, hd, nh, nkv = self.d, self.hd, self.nh, self.nkv
        group = nh // nkv
        x = self.w["embed"][int(token)].astype(np.float32).copy()
        cos, sin = self.cos[self.pos], self.sin[self.pos]
        for li, lw in enumerate(self.w["layers"]):
            xn = rmsnorm(x, lw["attn_norm"], self.eps)
            q = orc.gemv_bf16(lw["q"]["bits"], xn).reshape(nh, hd)
            kk = orc.gemv_bf16(lw["k"]["bits"], xn).reshape(nkv, hd)
            vv = orc.gemv_bf16(lw["v"]["bits"], xn).reshape(nkv, hd)
            q = rope(q, cos, sin)
            self.kc[li][:, self.pos] = orc.round_bf16(rope(kk, cos, sin))   # the cache holds bf16
            self.vc[li][:, self.pos] = orc.round_bf16(vv)
            attn = np.empty((nh, hd), np.float32)
            for h in range(nh):
                ks = self.kc[li][h // group, : self.pos + 1].astype(np.float64)
                vs = self.vc[li][h // group, : self.pos + 1].astype(np.float64)
                sc = (ks @ q[h].astype(np.float64)) / np.sqrt(hd)
                p = np.exp(sc - sc.max())
                attn[h] = ((p / p.sum()) @ vs).astype(np.float32)
            x = (x + orc.gemv_bf16(lw["o"]["bits"], attn.reshape(-1))).astype(np.float32)
            xn = rmsnorm(x, lw["ffn_norm"], self.eps)
            g = orc.gemv_bf16(lw["gate"]["bits"], xn)
            u = orc.gemv_bf16(lw["up"]["bits"], xn)
            act = (g / (np.float32(1.0) + np.exp(-g.astype(np.float32))) * u).astype(np.float32)
            x = (x + orc.gemv_bf16(lw["down"]["bits"], act)).astype(np.float32)
        xn = rmsnorm(x, self.w["final_norm"], self.eps)
        logits = orc.gemv_bf16(orc.to_bf16_bits(self.w["lm_head"]), xn)
        self.pos += 1
        return orc.argmax(logits), logits, x
