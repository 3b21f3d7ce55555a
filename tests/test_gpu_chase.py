"""Fused switch + GEMV ("chase" mode, include/adafuse_b200.h `af_switch_gemv`): one pass over a
projection's weights merges the selected experts (adapters.py:236-258 -> linalg.py:306-346) and
multiplies the merged, rounded tiles with the projection's input (model.py:288).

Checked here: the weights it leaves behind are BIT-IDENTICAL to the plain fused switch; the
accumulated outputs equal W_new . x (f64 on the host from the GPU's own bf16 bits) to f32
round-off; prologues (RMSNorm, SiLU*up, residual) follow the separate GEMV path; ragged shapes;
the result does not depend on CTA arrival order (bit-reproducible)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

FIX = 2.0 ** -40


@pytest.fixture(scope="module")
def af():
    import paper_2603_11873_b200 as af

    return af


def _bf16_to_f64(t):
    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)


def _mk_table(af, shapes, n_experts=6, rank=8, seed=0, pristine=False):
    from paper_2603_11873_b200.adapters import SwitchTable
    from paper_2603_11873_b200.linalg import Matrix

    g = torch.Generator(device="cuda").manual_seed(seed)

    def u(shape, fan):
        return (torch.empty(shape, device="cuda").uniform_(-1, 1, generator=g) * fan ** -0.5).to(torch.bfloat16)

    targets = [Matrix(u((o, i), i), "bf16") for o, i in shapes]
    downs = [u((n_experts, rank, i), i) for o, i in shapes]
    ups = [u((n_experts, o, rank), rank) for o, i in shapes]
    pr = [t.copy() for t in targets] if pristine else None
    return targets, SwitchTable(targets, downs, ups, pristine=pr)


def _decision(af, ids, weights):
    from paper_2603_11873_b200.routing import DeviceDecision, GateDecision

    return DeviceDecision.from_host(GateDecision(tuple(ids), tuple(weights)), torch.device("cuda"))


@pytest.mark.parametrize("d_in,rows", [(256, (64, 32, 32)), (1000, (96, 40, 72)), (520, (33,)), (2048, (512, 128, 128))])
@pytest.mark.parametrize("rank", [8, 16])
def test_switch_gemv_weights_and_outputs(af, d_in, rows, rank):
    from paper_2603_11873_b200.adapters import SegmentGroup

    shapes = [(r, d_in) for r in rows]
    tg_a, tab_a = _mk_table(af, shapes, rank=rank, seed=3)
    tg_b, tab_b = _mk_table(af, shapes, rank=rank, seed=3)
    for a, b in zip(tg_a, tg_b):
        assert torch.equal(a.data, b.data)
    prev = _decision(af, (1, 4), (0.7, 0.3))
    cur = _decision(af, (4, 2), (0.55, 0.45))
    grp = SegmentGroup(tab_a, range(len(shapes)))
    assert grp.x_len == d_in and grp.y_rows == sum(rows)
    x = torch.empty(d_in, device="cuda").uniform_(-1, 1)
    # merge prev (plain switch on both), then the steady step: fused on A, separate on B
    tab_a.switch(None, prev, max_k=2)
    tab_b.switch(None, prev, max_k=2)
    acc = torch.zeros(grp.y_rows, dtype=torch.int64, device="cuda")
    grp.switch_gemv(prev, cur, acc, xin=x, max_k=2)
    tab_b.switch(prev, cur, max_k=2)
    tab_a.status()
    # Same kernel family on both sides -> the same bits.  Between 33 and 64 stacked ranks the plain switch runs on
    # tcgen05 and the fused launch on mma.sync (af_api.cu kUmmaMaxRanks / kUmmaMaxRanksChain): the f32 sums differ in
    # order, so a rounding may tip on a rare element -- never more than one bf16 step.
    same_path = 4 * rank <= 32 or not tab_a.info()["umma_path"]
    for a, b in zip(tg_a, tg_b):
        if same_path:
            assert torch.equal(a.data, b.data), "fused switch + GEMV must leave the same weights as the plain switch"
        else:
            fa, fb = a.data.float(), b.data.float()
            mag = torch.maximum(torch.maximum(fa.abs(), fb.abs()), fa.abs().mean())     # cancellation: judge at the operands' size
            step = torch.exp2(torch.floor(torch.log2(mag)) - 7)
            assert ((fa - fb).abs() <= step).all() and (fa != fb).float().mean().item() < 1e-3
    w_new = np.concatenate([_bf16_to_f64(t.data) for t in tg_a], axis=0)
    want = w_new @ x.cpu().numpy().astype(np.float64)
    got = acc.cpu().numpy().astype(np.float64) * FIX
    scale = np.abs(w_new) @ np.abs(x.cpu().numpy().astype(np.float64))
    # x enters as bf16 hi + lo (2^-17 relative), products are exact, f32 accumulation per strip
    assert np.max(np.abs(got - want) / (scale + 1e-30)) < 2e-5
    # arrival-order independence: repeat from the same state, bit-identical accumulators
    acc2 = torch.zeros_like(acc)
    w_before = [a.data.clone() for a in tg_a]
    grp.switch_gemv(cur, cur, acc2, xin=x, max_k=2)       # unchanged decision: pure GEMV, nothing stored
    for a, b in zip(tg_a, w_before):
        assert torch.equal(a.data, b)
    assert torch.equal(acc, acc2)
    acc3 = torch.zeros_like(acc)
    grp.switch_gemv(None, None, acc3, xin=x)              # no decision at all: plain GEMV
    # (a launch without a decision may run on the other tensor path -- the tcgen05 kernel takes launches of up
    #  to 32 stacked ranks -- which sums a row in a different order: equal to f32 round-off, bitwise only when
    #  both launches are on one path)
    got3 = acc3.cpu().numpy().astype(np.float64) * FIX
    assert np.max(np.abs(got3 - got) / (scale + 1e-30)) < 2e-5
    if 4 * rank <= 32 or not tab_a.info()["umma_path"]:
        assert torch.equal(acc, acc3)


def test_switch_gemv_prologues(af):
    from paper_2603_11873_b200 import _capi
    from paper_2603_11873_b200.adapters import SegmentGroup
    from paper_2603_11873_b200.linalg import _ptr

    d_in, rows = 768, (160, 96)
    tg, tab = _mk_table(af, [(r, d_in) for r in rows], seed=5)
    grp = SegmentGroup(tab, [0, 1])
    cur = _decision(af, (0, 3), (0.6, 0.4))
    g = torch.Generator(device="cuda").manual_seed(9)
    acc_in = (torch.empty(2 * d_in, device="cuda").uniform_(-2, 2, generator=g) / FIX).to(torch.int64)
    res = torch.empty(d_in, device="cuda").uniform_(-1, 1, generator=g)
    nw = 1.0 + 0.1 * torch.empty(d_in, device="cuda").uniform_(-1, 1, generator=g)
    a = acc_in.cpu().numpy().astype(np.float64) * FIX
    # RMSNorm over h = res + fix(acc_in), h materialised
    acc = torch.zeros(grp.y_rows, dtype=torch.int64, device="cuda")
    h_out = torch.zeros(d_in, device="cuda")
    grp.switch_gemv(None, cur, acc, acc_in=acc_in, res=res, h_out=h_out, prologue="rmsnorm", norm_w=nw, eps=1e-5, max_k=2)
    w_new = np.concatenate([_bf16_to_f64(t.data) for t in tg], axis=0)
    h = res.cpu().numpy().astype(np.float64) + a[:d_in]
    np.testing.assert_allclose(h_out.cpu().numpy(), h, rtol=1e-6, atol=1e-6)
    xn = h / np.sqrt(np.mean(h * h) + 1e-5) * nw.cpu().numpy().astype(np.float64)
    got = acc.cpu().numpy().astype(np.float64) * FIX
    np.testing.assert_allclose(got, w_new @ xn, rtol=0, atol=3e-5 * np.max(np.abs(w_new) @ np.abs(xn)))
    # SiLU(gate) * up over the 2 * d_in accumulators; unchanged decision -> weights untouched
    acc.zero_()
    grp.switch_gemv(cur, cur, acc, acc_in=acc_in, prologue="silu_mul", max_k=2)
    xs = a[:d_in] / (1.0 + np.exp(-a[:d_in])) * a[d_in:]
    got = acc.cpu().numpy().astype(np.float64) * FIX
    np.testing.assert_allclose(got, w_new @ xs, rtol=0, atol=3e-5 * np.max(np.abs(w_new) @ np.abs(xs)))
    # hand-over kernel
    out = torch.zeros(d_in, device="cuda")
    _capi.check(_capi.lib().af_accum_to_f32(_ptr(acc_in), _ptr(res), _ptr(out), d_in, _capi.stream_ptr()))
    np.testing.assert_allclose(out.cpu().numpy(), h, rtol=1e-6, atol=1e-6)


def test_chain_equals_separate_launches(af):
    """o -> gate|up -> down -> q|k|v shaped chain in ONE launch (in-kernel phase barriers) against the
    same four projections launched one by one: bit-identical accumulators, residual streams, weights."""
    from paper_2603_11873_b200.adapters import SegmentGroup

    d, f = 512, 1280
    shapes = [(d, d), (f, d), (f, d), (d, f), (d, d), (128, d), (128, d)]      # o | gate up | down | q k v
    phases_ids = [[0], [1, 2], [3], [4, 5, 6]]
    outs = []
    for chained in (True, False):
        tg, tab = _mk_table(af, shapes, seed=7)
        prev = _decision(af, (1, 4), (0.7, 0.3))
        cur = _decision(af, (4, 2), (0.55, 0.45))
        tab.switch(None, prev, max_k=2)
        g = torch.Generator(device="cuda").manual_seed(2)
        attn = torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        xa = torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        nw1 = 1.0 + 0.1 * torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        nw2 = 1.0 + 0.1 * torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        xb, xa2 = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
        acc = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (d, 2 * f, d, d + 256)]
        phases = [dict(acc_out=acc[0], xin=attn),
                  dict(acc_out=acc[1], acc_in=acc[0], res=xa, h_out=xb, prologue="rmsnorm", norm_w=nw1, eps=1e-5),
                  dict(acc_out=acc[2], acc_in=acc[1], prologue="silu_mul"),
                  dict(acc_out=acc[3], acc_in=acc[2], res=xb, h_out=xa2, prologue="rmsnorm", norm_w=nw2, eps=1e-5)]
        if chained:
            done = torch.zeros(4, dtype=torch.int32, device="cuda")
            grp = SegmentGroup(tab, phases_ids)
            assert grp.n_phases == 4 and grp.x_lens == [d, d, f, d]
            grp.switch_gemv_chain(prev, cur, phases, done, max_k=2)
            torch.cuda.synchronize()
            counts = done[:3].tolist()          # every CTA of the launch published every phase
            assert counts[0] > 0 and counts == [counts[0]] * 3
        else:
            for ids, ph in zip(phases_ids, phases):
                SegmentGroup(tab, ids).switch_gemv_chain(prev, cur, [ph], None, max_k=2)
        tab.status()
        outs.append(([a.clone() for a in acc], xb.clone(), xa2.clone(), [t.data.clone() for t in tg]))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert torch.equal(a, b)
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])
    for a, b in zip(outs[0][3], outs[1][3]):
        assert torch.equal(a, b)
    assert float(outs[0][0][3].abs().max()) > 0


def test_weighted_schedule_changes_nothing_but_the_split(af):
    """af_chain_create_weighted: per-CTA shares of each phase (what `LlamaEngine.calibrate_schedule` measures) move
    tiles between CTAs; weights, accumulators and residual streams stay bit-identical to the equal split."""
    from paper_2603_11873_b200 import _capi
    from paper_2603_11873_b200.adapters import SegmentGroup

    d, f = 512, 1280
    shapes = [(d, d), (f, d), (f, d), (d, f), (d, d), (128, d), (128, d)]
    phases_ids = [[0], [1, 2], [3], [4, 5, 6]]
    n_cta = _capi.device_info()["sm_count"]
    rng = np.random.Generator(np.random.PCG64(5))
    outs = []
    for weighted in (False, True):
        tg, tab = _mk_table(af, shapes, seed=7)
        prev = _decision(af, (1, 4), (0.7, 0.3))
        cur = _decision(af, (4, 2), (0.55, 0.45))
        tab.switch(None, prev, max_k=2)
        g = torch.Generator(device="cuda").manual_seed(2)
        attn = torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        xa = torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        nw1 = 1.0 + 0.1 * torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        nw2 = 1.0 + 0.1 * torch.empty(d, device="cuda").uniform_(-1, 1, generator=g)
        xb, xa2 = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
        acc = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (d, 2 * f, d, d + 256)]
        phases = [dict(acc_out=acc[0], xin=attn),
                  dict(acc_out=acc[1], acc_in=acc[0], res=xa, h_out=xb, prologue="rmsnorm", norm_w=nw1, eps=1e-5),
                  dict(acc_out=acc[2], acc_in=acc[1], prologue="silu_mul"),
                  dict(acc_out=acc[3], acc_in=acc[2], res=xb, h_out=xa2, prologue="rmsnorm", norm_w=nw2, eps=1e-5)]
        share = rng.uniform(0.5, 1.5, (4, n_cta)).tolist() if weighted else None
        grp = SegmentGroup(tab, phases_ids, cta_share=share)
        done = torch.zeros(4, dtype=torch.int32, device="cuda")
        grp.switch_gemv_chain(prev, cur, phases, done, max_k=2)
        tab.status()
        outs.append(([a.clone() for a in acc], xb.clone(), xa2.clone(), [t.data.clone() for t in tg]))
    for a, b in zip(outs[0][0], outs[1][0]):
        assert torch.equal(a, b)
    assert torch.equal(outs[0][1], outs[1][1]) and torch.equal(outs[0][2], outs[1][2])
    for a, b in zip(outs[0][3], outs[1][3]):
        assert torch.equal(a, b)
    tg, tab = _mk_table(af, shapes, seed=7)
    with pytest.raises(ValueError):
        SegmentGroup(tab, phases_ids, cta_share=[[1.0] * n_cta] * 3 + [[0.0] * n_cta])


def test_group_validation(af):
    from paper_2603_11873_b200.adapters import SegmentGroup
    from paper_2603_11873_b200.errors import AliasingError, DimensionError

    tg, tab = _mk_table(af, [(64, 256), (64, 512)], seed=1)
    with pytest.raises(DimensionError):
        SegmentGroup(tab, [0, 1])            # different d_in: no shared input vector
    with pytest.raises(AliasingError):
        SegmentGroup(tab, [0, 0])
    with pytest.raises(IndexError):
        SegmentGroup(tab, [2])
    grp = SegmentGroup(tab, [1])
    acc = torch.zeros(64, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        grp.switch_gemv(None, None, acc)     # neither xin nor acc_in
    with pytest.raises(DimensionError):
        grp.switch_gemv(None, None, acc[:10], xin=torch.zeros(512, device="cuda"))


def test_chase_engine_equals_separate_engine(af):
    """Whole decode steps: the one-pass engine leaves bit-identical weights and the same tokens as
    switch-then-forward; logits agree to f32 round-off of the different summation orders."""
    from paper_2603_11873_b200 import llama

    forced = np.random.Generator(np.random.PCG64(21)).integers(0, 512, 12)
    engs = {}
    for mode in ("chase", "separate", "chase-unchained"):
        e = llama.LlamaEngine(llama.preset("tiny", max_seq=32, forward_mode=mode.split("-")[0], chain=(mode == "chase")), init="host")
        e.reset(forced=forced)
        lg = []
        for _ in range(12):
            e.decode_step()
            lg.append(e.logits.cpu().numpy().copy())
        engs[mode] = (e, np.stack(lg))
    (a, la), (b, lb) = engs["chase"], engs["separate"]
    assert a.chase and not b.chase
    for ta, tb in zip(a.targets, b.targets):
        assert torch.equal(ta.data, tb.data)
    np.testing.assert_allclose(la, lb, rtol=0, atol=2e-4 * np.max(np.abs(lb)))
    assert a.tokens() == b.tokens()
    c, lc = engs["chase-unchained"]
    assert c.chase and not c.chase_chained and a.chase_chained
    assert np.array_equal(la, lc)            # chaining is a schedule change only: bit-identical logits
    a.finalize()
    assert a.max_backbone_deviation() < 0.02


def test_deferred_rmsnorm_scale(af):
    """AF_PRO_RMSNORM_DEFERRED (tcgen05 path): the launch multiplies by x * norm_w only; the scale
    rsqrt(mean(x^2) + eps) lands in inv_out and the consumer applies it -- inv_out * outputs equals the
    plain RMSNorm launch, and a SiLU phase given inv_in equals one fed pre-scaled accumulators."""
    from paper_2603_11873_b200.adapters import SegmentGroup

    d_in, rows = 512, (256, 128)
    tg, tab = _mk_table(af, [(r, d_in) for r in rows], seed=11)
    if not tab.info()["umma_path"]:
        pytest.skip("tcgen05 path not enabled")
    grp = SegmentGroup(tab, [0, 1])
    cur = _decision(af, (0, 3), (0.6, 0.4))
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.empty(d_in, device="cuda").uniform_(-3, 3, generator=g)
    nw = 1.0 + 0.1 * torch.empty(d_in, device="cuda").uniform_(-1, 1, generator=g)
    acc_plain = torch.zeros(grp.y_rows, dtype=torch.int64, device="cuda")
    acc_def = torch.zeros_like(acc_plain)
    inv = torch.zeros(1, device="cuda")
    grp.switch_gemv(None, cur, acc_plain, xin=x, prologue="rmsnorm", norm_w=nw, eps=1e-5, max_k=2)
    grp.switch_gemv(cur, cur, acc_def, xin=x, prologue="rmsnorm_deferred", norm_w=nw, eps=1e-5, inv_out=inv, max_k=2)
    tab.status()
    want_inv = float(1.0 / np.sqrt(np.mean(x.cpu().numpy().astype(np.float64) ** 2) + 1e-5))
    assert abs(float(inv.item()) - want_inv) <= 1e-6 * want_inv
    a = acc_plain.cpu().numpy().astype(np.float64) * FIX
    b = acc_def.cpu().numpy().astype(np.float64) * FIX * float(inv.item())
    np.testing.assert_allclose(b, a, rtol=0, atol=3e-5 * np.max(np.abs(a)))
    # consumer side: SiLU(gate) * up over accumulators that still lack the scale
    tg2, tab2 = _mk_table(af, [(128, 256)], seed=12)
    grp2 = SegmentGroup(tab2, [0])
    raw = (torch.empty(512, device="cuda").uniform_(-2, 2, generator=g) / FIX).to(torch.int64)
    scale = torch.full((1,), 0.37, device="cuda")
    scaled = (raw.to(torch.float64) * 0.37).round().to(torch.int64)
    o1 = torch.zeros(128, dtype=torch.int64, device="cuda")
    o2 = torch.zeros_like(o1)
    grp2.switch_gemv(None, None, o1, acc_in=raw, prologue="silu_mul", inv_in=scale)
    grp2.switch_gemv(None, None, o2, acc_in=scaled, prologue="silu_mul")
    v1, v2 = o1.cpu().numpy() * FIX, o2.cpu().numpy() * FIX
    np.testing.assert_allclose(v1, v2, rtol=0, atol=2e-5 * np.max(np.abs(v2)))
