"""Unit parity of the bs=1 decode kernels through the C ABI: fused GEMV (prologues, epilogues,
both streaming variants), the toy-stack GEMV / transposed GEMV / argmax, and decode attention
(RoPE + KV append + GQA, split over CTAs) against numpy restatements."""

import ctypes

import numpy as np
import pytest
import torch

from oracle import llama_oracle as lo
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def capi():
    from paper_2603_11873_b200 import _capi

    return _capi


def _dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda().to(dtype)


@pytest.mark.parametrize("variant", [0, 1, 4])
@pytest.mark.parametrize("rows,cols", [(64, 256), (300, 1024), (4096, 4096), (1000, 11008), (7, 8)])
def test_gemv_fused_prologues_and_epilogues(capi, variant, rows, cols):
    L = capi.lib()
    capi.check(L.af_set_gemv_variant(variant, 0))
    rng = np.random.Generator(np.random.PCG64(rows * 7 + cols))
    w = orc.round_bf16(rng.uniform(-1, 1, (rows, cols)).astype(np.float32) / np.sqrt(cols))
    wd = _dev(w, torch.bfloat16)
    st = capi.stream_ptr()
    x = rng.normal(size=cols).astype(np.float32)
    res = rng.normal(size=rows).astype(np.float32)
    nw = (1 + 0.1 * rng.normal(size=cols)).astype(np.float32)
    xu = rng.normal(size=2 * cols).astype(np.float32)
    out = torch.zeros(rows, dtype=torch.float32, device="cuda")
    xd, resd, nwd, xud = _dev(x), _dev(res), _dev(nw), _dev(xu)      # keep the device buffers alive across the async launches
    # (1) plain + residual epilogue
    capi.check(L.af_gemv_fused(wd.data_ptr(), rows, cols, cols, xd.data_ptr(), out.data_ptr(), capi.AF_PRO_NONE, None, 0.0,
                               capi.AF_EPI_RESIDUAL, resd.data_ptr(), st))
    want = res + orc.gemv_bf16(orc.to_bf16_bits(w), x)
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=2e-5, atol=2e-5)
    # (2) RMSNorm prologue
    capi.check(L.af_gemv_fused(wd.data_ptr(), rows, cols, cols, xd.data_ptr(), out.data_ptr(), capi.AF_PRO_RMSNORM, nwd.data_ptr(),
                               1e-5, capi.AF_EPI_NONE, None, st))
    want = orc.gemv_bf16(orc.to_bf16_bits(w), lo.rmsnorm(x, nw, 1e-5))
    np.testing.assert_allclose(out.cpu().numpy(), want, rtol=1e-4, atol=1e-4)
    # (3) SiLU(gate) * up prologue + GELU-residual epilogue (model.py:298-305)
    capi.check(L.af_gemv_fused(wd.data_ptr(), rows, cols, cols, xud.data_ptr(), out.data_ptr(), capi.AF_PRO_SILU_MUL, None, 0.0,
                               capi.AF_EPI_GELU_RESIDUAL, resd.data_ptr(), st))
    g, u = xu[:cols], xu[cols:]
    y = orc.gemv_bf16(orc.to_bf16_bits(w), (g / (1 + np.exp(-g)) * u).astype(np.float32))
    np.testing.assert_allclose(out.cpu().numpy(), orc.gelu_residual(y, res), rtol=2e-4, atol=2e-4)
    capi.check(L.af_set_gemv_variant(0, 0))


def test_gemv_fused_errors(capi):
    L = capi.lib()
    w = torch.zeros((8, 16), dtype=torch.bfloat16, device="cuda")
    x = torch.zeros(16, device="cuda")
    o = torch.zeros(8, device="cuda")
    st = capi.stream_ptr()
    assert L.af_gemv_fused(w.data_ptr(), 8, 12, 12, x.data_ptr(), o.data_ptr(), 0, None, 0.0, 0, None, st) == capi.AF_EDIM
    assert L.af_gemv_fused(w.data_ptr(), 8, 16, 16, x.data_ptr(), o.data_ptr(), 7, None, 0.0, 0, None, st) == capi.AF_EVALUE
    assert L.af_gemv_fused(w.data_ptr(), 8, 16, 16, x.data_ptr(), o.data_ptr(), capi.AF_PRO_RMSNORM, None, 0.0, 0, None, st) == capi.AF_EVALUE
    assert L.af_gemv_fused(w.data_ptr(), 8, 16, 16, x.data_ptr(), o.data_ptr(), 0, None, 0.0, capi.AF_EPI_RESIDUAL, None, st) == capi.AF_EVALUE
    assert L.af_gemv_fused(w.data_ptr(), 8, 16, 16, x.data_ptr(), x.data_ptr(), 0, None, 0.0, 0, None, st) == capi.AF_EALIAS


@pytest.mark.parametrize("dtype", ["bf16", "single"])
def test_toy_stack_kernels(dtype):
    import paper_2603_11873_b200 as af

    rng = np.random.Generator(np.random.PCG64(3))
    for rows, cols in [(256, 256), (33, 70), (1000, 64)]:
        w = orc.round_bf16(rng.uniform(-1, 1, (rows, cols)).astype(np.float32))
        x = rng.normal(size=(cols, 1)).astype(np.float32)
        rec = af.DispatchRecorder()
        y = af.gemm(af.Matrix(w, dtype), af.Matrix(x, "single"), rec, label="backbone")
        np.testing.assert_allclose(y.numpy()[:, 0], orc.gemv(w, x), rtol=1e-5, atol=1e-5)
        r = rng.normal(size=(rows, 1)).astype(np.float32)
        y2 = af.gemm(af.Matrix(w, dtype), af.Matrix(x, "single"), rec, epilogue="gelu_residual", residual=af.Matrix(r, "single"))
        np.testing.assert_allclose(y2.numpy()[:, 0], orc.gelu_residual(orc.gemv(w, x), r[:, 0]), rtol=1e-4, atol=1e-5)
        xt = rng.normal(size=(1, rows)).astype(np.float32)
        z = af.gemm(af.Matrix(xt, "single"), af.Matrix(w, dtype), rec)           # model.py:261-263 `_unembed`
        np.testing.assert_allclose(z.numpy()[0], orc.unembed(w, xt[0]), rtol=1e-5, atol=1e-5)
        assert [e.kind for e in rec.events] == ["gemm"] * 3
        assert rec.events[0].flops == 2 * rows * cols
    with pytest.raises(af.DimensionError):
        af.gemm(af.Matrix(np.zeros((4, 4)), "single"), af.Matrix(np.zeros((4, 3)), "single"), af.DispatchRecorder())
    with pytest.raises(af.PrecisionError):
        af.gemm(af.Matrix(np.zeros((4, 4)), "single"), af.Matrix(np.zeros((4, 1)), "bf16"), af.DispatchRecorder())


def test_argmax_lowest_index_on_ties(capi):
    L = capi.lib()
    v = np.zeros(5000, np.float32)
    v[[4097, 123, 4999]] = 7.5
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    val = torch.zeros(1, dtype=torch.float32, device="cuda")
    vd = _dev(v)
    capi.check(L.af_argmax(vd.data_ptr(), v.size, out.data_ptr(), capi.stream_ptr()))
    assert int(out.item()) == 123 == orc.argmax(v)                                  # model.py:396
    capi.check(L.af_argmax_val(vd.data_ptr(), v.size, 1000, out.data_ptr(), val.data_ptr(), capi.stream_ptr()))
    assert int(out.item()) == 1123 and float(val.item()) == 7.5


@pytest.mark.parametrize("hd,n_heads,n_kv,splits", [(64, 4, 2, 1), (128, 8, 2, 1), (128, 8, 8, 3), (256, 2, 1, 2), (80, 4, 4, 1), (128, 32, 8, 5),
                                                    (128, 4, 2, 8)])
def test_attention_decode_against_numpy(capi, hd, n_heads, n_kv, splits):
    """The grid carries `splits` CTAs per head; the kernel uses ceil(positions / 32) of them, so the run crosses
    every change of the effective split count (the 8-split case runs to 170 positions: 1 -> 6 splits)."""
    L = capi.lib()
    steps = 170 if splits == 8 else 70
    max_seq, theta = (192 if splits == 8 else 96), 10000.0
    rng = np.random.Generator(np.random.PCG64(hd + n_heads))
    cos, sin = lo.rope_tables(hd, max_seq, theta)
    kc = torch.zeros((n_kv, max_seq, hd), dtype=torch.bfloat16, device="cuda")
    vc = torch.zeros_like(kc)
    kc_ref = np.zeros((n_kv, max_seq, hd), np.float32)
    vc_ref = np.zeros_like(kc_ref)
    out = torch.zeros(n_heads * hd, dtype=torch.float32, device="cuda")
    pos = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = torch.zeros(n_heads * splits * (hd + 2), dtype=torch.float32, device="cuda")
    tickets = torch.zeros(n_heads, dtype=torch.int32, device="cuda")
    group = n_heads // n_kv
    cosd, sind = _dev(cos), _dev(sin)
    qkvd = torch.zeros((n_heads + 2 * n_kv) * hd, dtype=torch.float32, device="cuda")
    for t in range(steps):
        qkv = rng.normal(size=(n_heads + 2 * n_kv) * hd).astype(np.float32)
        pos.fill_(t)
        qkvd.copy_(torch.from_numpy(qkv))
        capi.check(L.af_attn_decode(qkvd.data_ptr(), kc.data_ptr(), vc.data_ptr(), cosd.data_ptr(), sind.data_ptr(),
                                    pos.data_ptr(), n_heads, n_kv, hd, max_seq, splits, ws.data_ptr(), tickets.data_ptr(),
                                    out.data_ptr(), capi.stream_ptr()))
        q = lo.rope(qkv[: n_heads * hd].reshape(n_heads, hd), cos[t], sin[t])
        k = qkv[n_heads * hd: (n_heads + n_kv) * hd].reshape(n_kv, hd)
        v = qkv[(n_heads + n_kv) * hd:].reshape(n_kv, hd)
        kc_ref[:, t] = orc.round_bf16(lo.rope(k, cos[t], sin[t]))
        vc_ref[:, t] = orc.round_bf16(v)
        want = np.empty((n_heads, hd), np.float32)
        for h in range(n_heads):
            sc = (kc_ref[h // group, : t + 1].astype(np.float64) @ q[h].astype(np.float64)) / np.sqrt(hd)
            p = np.exp(sc - sc.max())
            want[h] = (p / p.sum()) @ vc_ref[h // group, : t + 1].astype(np.float64)
        if t in (0, 1, 7, 8, 31, 32, 33, 63, 64, 69, 95, 96, 127, 128, 159, 160, 169):
            np.testing.assert_allclose(out.cpu().numpy().reshape(n_heads, hd), want, rtol=2e-4, atol=2e-5)
    # the cache holds the bf16-rounded rotated keys (the GPU contracts x*c - y*s into an FMA, so a value
    # on a rounding boundary may land on the neighbouring bf16: at most 1 ulp, a handful of elements)
    got_bits = kc[:, :steps].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    worst, ndiff = orc.max_ulp_diff_bf16(got_bits, orc.to_bf16_bits(kc_ref[:, :steps]))
    assert worst <= 1 and ndiff <= got_bits.size // 1000 + 1
    np.testing.assert_array_equal(vc.float().cpu().numpy()[:, :steps], vc_ref[:, :steps])
    assert int(tickets.sum().item()) == 0                                              # tickets reset for graph replay


@pytest.mark.parametrize("d,f,kv,vocab", [(256, 512, 128, 520), (1000, 2760, 200, 333), (4096, 11008, 4096, 2048)])
def test_gemv_chain_against_numpy(capi, d, f, kv, vocab):
    """o -> gate|up -> down -> q|k|v (and -> lm_head-like) as one persistent launch (af_gemv_chain):
    each phase against the numpy restatement fed with the GPU's own previous-phase outputs."""
    L = capi.lib()
    st = capi.stream_ptr()
    rng = np.random.Generator(np.random.PCG64(d + f))

    def mk(rows, cols):
        w = orc.round_bf16(rng.uniform(-1, 1, (rows, cols)).astype(np.float32) / np.sqrt(cols))
        return w, _dev(w, torch.bfloat16)

    wo, wo_d = mk(d, d)
    wgu, wgu_d = mk(2 * f, d)
    wdn, wdn_d = mk(d, f)
    wq, wq_d = mk(d + 2 * kv, d)
    attn = rng.normal(size=d).astype(np.float32)
    xa = rng.normal(size=d).astype(np.float32)
    nw1 = (1 + 0.1 * rng.normal(size=d)).astype(np.float32)
    nw2 = (1 + 0.1 * rng.normal(size=d)).astype(np.float32)
    attn_d, xa_d, nw1_d, nw2_d = _dev(attn), _dev(xa), _dev(nw1), _dev(nw2)
    xb_d = torch.zeros(d, device="cuda")
    gu_d = torch.zeros(2 * f, device="cuda")
    xa2_d = torch.zeros(d, device="cuda")
    qkv_d = torch.zeros(d + 2 * kv, device="cuda")
    P = capi.GvPhase
    p = lambda t: t.data_ptr()  # noqa: E731
    phases = (P * 4)(
        P(w=p(wo_d), rows=d, cols=d, ld=d, x=p(attn_d), out=p(xb_d), res=p(xa_d), norm_w=None, eps=0.0, prologue=capi.AF_PRO_NONE,
          epilogue=capi.AF_EPI_RESIDUAL),
        P(w=p(wgu_d), rows=2 * f, cols=d, ld=d, x=p(xb_d), out=p(gu_d), res=None, norm_w=p(nw1_d), eps=1e-5, prologue=capi.AF_PRO_RMSNORM,
          epilogue=capi.AF_EPI_NONE),
        P(w=p(wdn_d), rows=d, cols=f, ld=f, x=p(gu_d), out=p(xa2_d), res=p(xb_d), norm_w=None, eps=0.0, prologue=capi.AF_PRO_SILU_MUL,
          epilogue=capi.AF_EPI_RESIDUAL),
        P(w=p(wq_d), rows=d + 2 * kv, cols=d, ld=d, x=p(xa2_d), out=p(qkv_d), res=None, norm_w=p(nw2_d), eps=1e-5,
          prologue=capi.AF_PRO_RMSNORM, epilogue=capi.AF_EPI_NONE),
    )
    done = torch.zeros(4, dtype=torch.int32, device="cuda")
    capi.check(L.af_gemv_chain(phases, 4, p(done), None, 0, st))
    torch.cuda.synchronize()
    sm = capi.device_info()["sm_count"]
    assert done[:3].tolist() == [sm] * 3
    xb = xb_d.cpu().numpy()
    np.testing.assert_allclose(xb, xa + orc.gemv_bf16(orc.to_bf16_bits(wo), attn), rtol=2e-5, atol=2e-5)
    gu = gu_d.cpu().numpy()
    np.testing.assert_allclose(gu, orc.gemv_bf16(orc.to_bf16_bits(wgu), lo.rmsnorm(xb, nw1, 1e-5)), rtol=1e-4, atol=1e-4)
    g, u = gu[:f], gu[f:]
    xa2 = xa2_d.cpu().numpy()
    np.testing.assert_allclose(xa2, xb + orc.gemv_bf16(orc.to_bf16_bits(wdn), (g / (1 + np.exp(-g)) * u).astype(np.float32)),
                               rtol=2e-4, atol=2e-4)
    np.testing.assert_allclose(qkv_d.cpu().numpy(), orc.gemv_bf16(orc.to_bf16_bits(wq), lo.rmsnorm(xa2, nw2, 1e-5)), rtol=1e-4, atol=1e-4)
    # bit-reproducible: a second run from the same inputs gives the same bits
    q1 = qkv_d.clone()
    done.zero_()
    capi.check(L.af_gemv_chain(phases, 4, p(done), None, 0, st))
    torch.cuda.synchronize()
    assert torch.equal(q1, qkv_d)
    # validation
    with pytest.raises(ValueError):
        capi.check(L.af_gemv_chain(phases, 5, p(done), None, 0, st))
    with pytest.raises(ValueError):
        capi.check(L.af_gemv_chain(phases, 2, None, None, 0, st))
