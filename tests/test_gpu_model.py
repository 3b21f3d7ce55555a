"""Decode-engine parity on the GPU: the toy decoder stack of the reference (model.py) run
through the B200 path against (a) fixtures generated from the unmodified reference on
bf16-rounded weights and (b) the CPU oracle following the GPU's bf16 weights step by step."""

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def af():
    import paper_2603_11873_b200 as af

    return af


def _cfg(af, g, name, **kw):
    layers, hidden, vocab, experts, rank, top_k, seed = (int(v) for v in g[f"{name}_config"])
    return af.ModelConfig(layers=layers, hidden=hidden, vocab=vocab, experts=experts, rank=rank, top_k=top_k, seed=seed, **kw)


def test_weights_match_reference_draw(af, golden):
    # /root/reference/pkg/tests/test_model.py:30-33: one seed names one model
    import hashlib

    cfg = af.ModelConfig(layers=4, hidden=8, vocab=16, experts=4, rank=2, top_k=2, precision="single", seed=42)
    model = af.build_model(cfg)
    want = bytes(golden("generate")["digest_single_seed42"]).decode()
    assert af.weights_digest(model) == want
    assert len(want) == hashlib.sha256().digest_size * 2


@pytest.mark.parametrize("switch_mode,refresh_every", [("inplace", 0), ("from_pristine", 0), ("inplace", -1)],
                         ids=["inplace-default", "from_pristine", "inplace-never-refreshed"])
@pytest.mark.parametrize("name", ["small", "c1", "c1v1024"])
def test_forced_stream_against_reference(af, golden, name, switch_mode, refresh_every):
    """Teacher-forced decode: router ids bit-exact, next tokens identical, logits <= 1e-2
    relative on EVERY step of the 64-token stream, all against the reference running f32
    arithmetic on the same bf16 weights (north_star's criterion, no widened band).

    The reference keeps the live weights in f32; bf16 storage re-rounds W at every in-place
    switch (a ~0.3*sqrt(T) ulp random walk).  The default in-place bf16 model
    therefore rebuilds W from the pristine copy every 16 tokens (model.py:344-349 `refresh_every`,
    folded into that token's switch launch: `ModelConfig.effective_refresh_every`), and
    "from_pristine" never accumulates rounding at all.  The third variant turns the refresh off
    (refresh_every=-1) and documents what it is for: the band is checked for the first 16 switches only."""
    g = golden("generate")
    model = af.build_model(_cfg(af, g, name, switch_mode=switch_mode, refresh_every=refresh_every))
    assert model.config.effective_refresh_every == (16 if (switch_mode, refresh_every) == ("inplace", 0) else 0)
    forced = g[f"{name}_forced_tokens"]
    if refresh_every < 0:
        forced = forced[:16]
    state = af.DecodeState()
    rec = af.DispatchRecorder()
    n_layers = model.config.layers
    for step, tkn in enumerate(forced):
        logits = []
        nxt, events = af.decode_step(model, state, int(tkn), rec, logits_out=logits)
        dec = state.prev_decision.to_host()
        if g[f"{name}_forced_margin"][step] > 1e-6:
            assert dec.expert_ids == tuple(int(v) for v in g[f"{name}_forced_ids"][step]), f"step {step}"
            np.testing.assert_allclose(dec.weights, g[f"{name}_forced_weights"][step], rtol=1e-5)
        want = g[f"{name}_forced_logits"][step]
        scale = np.max(np.abs(want))
        band = 1e-2
        assert np.max(np.abs(logits[0] - want)) <= band * scale, f"step {step}"
        top2 = np.sort(want)[-2:]
        if top2[1] - top2[0] > 2 * band * scale:
            assert nxt == int(g[f"{name}_forced_next"][step])
        kinds = [e.kind for e in events]
        assert kinds.count("sgmm") == 1 and kinds.count("reduce") == 1      # tests/test_model.py:204-225
        assert kinds.count("gemm") == n_layers + 2
    af.finalize_generation(model, state, rec)
    assert state.prev_decision is None
    # bf16 storage re-rounds W every switch: residue is a few bf16 ulps of |W| <= 1/sqrt(d)
    assert af.max_backbone_deviation(model) < 0.01


@pytest.mark.parametrize("compute", ["exact", "auto"])
def test_forced_stream_against_oracle_stepwise(af, compute):
    """Per-step oracle on the GPU's own bf16 weights: decisions identical, merged W within
    1 bf16 ulp (bit-exact in EXACT order), hidden state and logits within 1e-2 relative."""
    cfg = af.ModelConfig(layers=4, hidden=256, vocab=256, experts=8, rank=8, top_k=2, seed=0, compute=compute)
    model = af.build_model(cfg)
    om = orc.build_toy_model(orc.ToyConfig(layers=4, hidden=256, vocab=256, experts=8, rank=8, top_k=2, seed=0,
                                           refresh_every=cfg.effective_refresh_every), bf16=True)
    for li in range(cfg.layers):
        assert np.array_equal(model.backbone[li].bits(), om.backbone_bits[li])
    forced = np.random.Generator(np.random.PCG64(1)).integers(0, cfg.vocab, 24)     # crosses the refresh at token 16
    state, ostate = af.DecodeState(), orc.ToyState()
    rec = af.DispatchRecorder()
    for step, tkn in enumerate(forced):
        logits = []
        before = [b.copy() for b in om.backbone_bits]
        prev_dec = ostate.prev
        nxt, _ = af.decode_step(model, state, int(tkn), rec, logits_out=logits)
        o_next, o_logits, o_dec = orc.toy_decode_step(om, ostate, int(tkn), storage="bf16")
        dec = state.prev_decision.to_host()
        assert dec.expert_ids == o_dec[0]
        np.testing.assert_allclose(dec.weights, o_dec[1], rtol=2e-6)
        for li in range(cfg.layers):
            got = model.backbone[li].bits()
            if compute == "exact":
                worst, ndiff = orc.max_ulp_diff_bf16(got, om.backbone_bits[li])
                assert worst == 0, f"step {step} layer {li}: {ndiff} diffs, max {worst} ulp"
            else:
                mid = before[li].copy()
                orc.switch_segment_bf16(mid, orc.to_bf16_bits(om.down_bank[li]), orc.to_bf16_bits(om.up_bank[li]), prev_dec, None)
                worst, ndiff = orc.merge_error_in_ulps(got, om.backbone_bits[li], before[li], mid)
                assert worst <= 1.0, f"step {step} layer {li}: {ndiff} diffs, max {worst} ulp"
            om.backbone_bits[li][...] = got              # oracle follows the GPU's live weights
        scale = np.max(np.abs(o_logits))
        assert np.max(np.abs(logits[0] - o_logits)) <= 1e-2 * scale
        np.testing.assert_allclose(state.last_hidden, ostate.last_hidden, rtol=1e-2, atol=1e-4)


def test_generate_api_and_restore(af, golden):
    g = golden("generate")
    model = af.build_model(_cfg(af, g, "small"))
    rec = af.DispatchRecorder()
    sink = []
    toks, trace = af.generate(model, [7, 42, 3], 16, rec, hidden_sink=sink)
    assert len(toks) == 16 and len(sink) == 16 and len(sink[0]) == model.config.layers
    from paper_2603_11873_b200.perf import DispatchTrace

    assert isinstance(trace, DispatchTrace) and len(trace.events) == len(trace)      # model.py:428-457 returns a DispatchTrace
    assert sum(1 for ev in trace if ev.kind == "sgmm") == int(g["small_sgmm_events"]) == 16
    want = g["small_greedy_hidden_last"]
    got = np.stack([s[-1] for s in sink])
    # greedy feedback is chaotic once a near-tie flips a token; compare until the streams part
    ref_toks = g["small_greedy_tokens"]
    same = 0
    while same < 16 and toks[same] == int(ref_toks[same]):
        same += 1
    assert same >= 1
    np.testing.assert_allclose(got[: same], want[: same], rtol=2e-2, atol=2e-3)
    assert af.max_backbone_deviation(model) < 0.01
    with pytest.raises(af.InputError):
        af.generate(model, [1], 0, rec)
    with pytest.raises(af.InputError):
        af.generate(model, [], 4, rec)
    with pytest.raises(af.InputError):
        af.decode_step(model, af.DecodeState(), model.config.vocab, rec)


def test_repeated_token_cancels_and_refresh_every(af):
    # tests/test_model.py:256-268, :367-381
    cfg = af.ModelConfig(layers=3, hidden=64, vocab=64, experts=4, rank=8, top_k=2, seed=5, refresh_every=3)
    model = af.build_model(cfg)
    state = af.DecodeState()
    rec = af.DispatchRecorder()
    af.decode_step(model, state, 9, rec)
    w_after_first = [m.bits().copy() for m in model.backbone]
    af.decode_step(model, state, 9, rec)                 # same token -> same decision -> no-op switch
    for m, w in zip(model.backbone, w_after_first):
        assert np.array_equal(m.bits(), w)
    for t in (1, 2, 3, 4, 5, 6):
        af.decode_step(model, state, t, rec)
    af.finalize_generation(model, state, rec)
    assert af.max_backbone_deviation(model) < 0.05


def test_base_strategy_and_simple_merge(af):
    cfg = af.ModelConfig(layers=3, hidden=64, vocab=64, experts=4, rank=8, top_k=2, seed=5, strategy=af.Strategy.BASE)
    model = af.build_model(cfg)
    rec = af.DispatchRecorder()
    toks, trace = af.generate(model, [3], 4, rec)
    assert not any(ev.kind == "sgmm" for ev in trace)
    assert af.max_backbone_deviation(model) == 0.0
    fused = af.build_model(af.ModelConfig(layers=3, hidden=64, vocab=64, experts=4, rank=8, top_k=2, seed=5))
    simple = af.build_model(af.ModelConfig(layers=3, hidden=64, vocab=64, experts=4, rank=8, top_k=2, seed=5,
                                           strategy=af.Strategy.PRE_GATED_SIMPLE_MERGE))
    sa, sb = af.DecodeState(), af.DecodeState()
    for t in (5, 9, 11, 2):
        la, lb = [], []
        af.decode_step(fused, sa, t, af.DispatchRecorder(), logits_out=la)
        af.decode_step(simple, sb, t, af.DispatchRecorder(), logits_out=lb)
        np.testing.assert_allclose(la[0], lb[0], rtol=2e-2, atol=2e-3)
