"""Llama-shaped engine on the GPU against the CPU restatement (oracle/llama_oracle.py):
router ids bit-exact, merged weights of all 7 x L segments within 1 bf16 ulp, logits within
1e-2 relative; eager steps == captured-graph steps; TP shards == slices of the full model."""

import numpy as np
import pytest
import torch

from oracle import llama_oracle as lo
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def llama():
    from paper_2603_11873_b200 import llama

    return llama


def _bits(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16).copy()


def _oracle_for(eng, llama):
    cfg = eng.cfg
    names = llama.SEGMENT_NAMES
    layers = []
    for li in range(cfg.layers):
        lw = {"attn_norm": eng.attn_norm[li].cpu().numpy(), "ffn_norm": eng.ffn_norm[li].cpu().numpy()}
        for j, name in enumerate(names):
            i = li * len(names) + j
            lw[name] = {"bits": _bits(eng.targets[i].data), "down": _bits(eng.bank_down[i]), "up": _bits(eng.bank_up[i])}
        layers.append(lw)
    w = {"embed": eng.embed.numpy(), "router": eng.router.numpy(), "lm_head": eng.lm_head.numpy(),
         "final_norm": eng.final_norm.cpu().numpy(), "layers": layers}
    return lo.LlamaOracle(w, hidden=cfg.hidden, n_heads=cfg.n_heads, n_kv_heads=cfg.n_kv_heads, top_k=cfg.top_k,
                          rope_theta=cfg.rope_theta, rms_eps=cfg.rms_eps, max_seq=cfg.max_seq)


@pytest.mark.parametrize("shape", ["r8", "r16-gqa", "r32-k4"])
@pytest.mark.parametrize("forward_mode", ["chase", "separate"])
@pytest.mark.parametrize("switch_mode", ["inplace", "from_pristine"])
def test_decode_steps_against_oracle(llama, switch_mode, forward_mode, shape):
    # "r16-gqa": BASELINE configs[2]-like -- 16 experts of rank 16, 4 query heads on 1 kv head
    # "r32-k4": BASELINE configs[4]-like -- rank 32, top-4: 256 stacked ranks in a steady switch, ONE K-chunked launch
    extra = {"r16-gqa": dict(experts=16, rank=16, n_heads=4, n_kv_heads=1), "r32-k4": dict(experts=8, rank=32, top_k=4)}.get(shape, {})
    cfg = llama.preset("tiny", switch_mode=switch_mode, max_seq=32, forward_mode=forward_mode, **extra)
    eng = llama.LlamaEngine(cfg, init="host")
    assert eng.table.info()["tensor_path"]
    assert eng.chase == (forward_mode == "chase")
    ora = _oracle_for(eng, llama)
    pristine = [{n: ora.w["layers"][li][n]["bits"].copy() for n in llama.SEGMENT_NAMES} for li in range(cfg.layers)]
    forced = np.random.Generator(np.random.PCG64(11)).integers(0, cfg.vocab, 10)
    eng.reset(forced=forced)
    for step, tkn in enumerate(forced):
        before = [{n: ora.w["layers"][li][n]["bits"].copy() for n in llama.SEGMENT_NAMES} for li in range(cfg.layers)]
        nxt = eng.decode_step()
        eng.table.status()
        ids, wts = ora.route(tkn)
        prev_dec = ora.prev
        dec = eng.decision()
        assert dec.expert_ids == ids, f"step {step}"
        np.testing.assert_allclose(dec.weights, wts, rtol=2e-6)
        ora.switch((ids, wts), from_pristine=(switch_mode == "from_pristine"), pristine=pristine)
        for li in range(cfg.layers):
            for j, name in enumerate(llama.SEGMENT_NAMES):
                got = _bits(eng.targets[li * 7 + j].data)
                ref_before = pristine[li][name] if switch_mode == "from_pristine" else before[li][name]
                mid = ref_before.copy()
                if switch_mode == "inplace":
                    seg = ora.w["layers"][li][name]
                    orc.switch_segment_bf16(mid, seg["down"], seg["up"], prev_dec, None)
                worst, nd = orc.merge_error_in_ulps(got, ora.w["layers"][li][name]["bits"], ref_before, mid)
                assert worst <= 1.0, f"step {step} layer {li} {name}: {nd} diffs, max {worst} ulp"
                ora.w["layers"][li][name]["bits"][...] = got      # oracle follows the GPU's live weights
        o_next, o_logits, o_hidden = ora.forward(tkn)
        got_logits = eng.logits.cpu().numpy()
        scale = np.max(np.abs(o_logits))
        assert np.max(np.abs(got_logits - o_logits)) <= 1e-2 * scale, f"step {step}"
        top2 = np.sort(o_logits)[-2:]
        if top2[1] - top2[0] > 2e-2 * scale:
            assert nxt == o_next
    assert eng.steps_done() == len(forced)
    eng.finalize()
    assert eng.max_backbone_deviation() < 0.02


@pytest.mark.parametrize("forward_mode", ["chase", "separate"])
def test_graph_replay_equals_eager(llama, forward_mode):
    cfg = llama.preset("tiny", max_seq=48, forward_mode=forward_mode)
    forced = np.random.Generator(np.random.PCG64(12)).integers(0, cfg.vocab, 20)
    a = llama.LlamaEngine(cfg, init="host")
    a.reset(forced=forced)
    for _ in range(20):
        a.decode_step(graph=False)      # eager launches (decode_step replays a captured graph by default)
    eager = a.tokens()
    b = llama.LlamaEngine(cfg, init="host")
    b.reset(forced=forced)
    b.decode_step()
    b.capture()
    for _ in range(19):
        b.replay()
    torch.cuda.synchronize()
    assert b.tokens() == eager
    for ta, tb in zip(a.targets, b.targets):
        assert torch.equal(ta.data, tb.data)


@pytest.mark.parametrize("forward_mode", ["chase", "separate"])
def test_split_attention_and_pdl_do_not_change_results(llama, forward_mode):
    """flash-decoding split over CTAs and programmatic dependent launch are schedule changes only."""
    from paper_2603_11873_b200 import _capi

    forced = np.random.Generator(np.random.PCG64(13)).integers(0, 512, 24)
    outs = []
    # 80 positions: the kernel uses up to ceil(80 / 32) = 3 of the grid's splits, so the split runs really split
    forced = np.random.Generator(np.random.PCG64(13)).integers(0, 512, 80)
    for splits, pdl in ((1, 1), (3, 1), (1, 0), (5, 0)):
        _capi.check(_capi.lib().af_set_pdl(pdl))
        eng = llama.LlamaEngine(llama.preset("tiny", max_seq=96, attn_splits=splits, forward_mode=forward_mode), init="host")
        eng.reset(forced=forced)
        logits = []
        for _ in range(80):
            eng.decode_step()
            logits.append(eng.logits.cpu().numpy().copy())
        outs.append((eng.tokens(), np.stack(logits)))
    _capi.check(_capi.lib().af_set_pdl(1))
    # Split attention reorders f32 sums (1e-7 on the attention output).  In the one-pass forward the
    # activations enter the tensor pipe as bf16 hi + lo pairs -- x is reproduced to 2^-18, by a
    # rounding that a 1e-7 change re-rolls -- so bf16 roundings of cached k/v flip more often and
    # the schedules drift apart faster (still 20x inside the 1e-2 logit criterion).  The plain forward has the same
    # mechanism one level down: the KV cache stores bf16, and a 1e-7 change of k or v flips the occasional rounding
    # (2^-9 of one cached element: a few 1e-5 on a logit over 80 positions).
    atol = 1e-4 if forward_mode == "separate" else 1e-3
    for toks, lg in outs[1:]:
        np.testing.assert_allclose(lg, outs[0][1], rtol=1e-4, atol=atol)
    assert outs[2][0] == outs[0][0]          # PDL on/off: bit-identical schedule-independent arithmetic
    assert np.array_equal(outs[2][1], outs[0][1])


@pytest.mark.parametrize("shape", ["mha-hd64", "gqa-hd64", "hd128"])
def test_persistent_forward_equals_chained_forward(llama, shape):
    """af_forward_persistent (the whole forward of a token -- attention included -- as ONE launch over a device-side
    phase table) against the chained forward with the standalone attention kernel: same tokens, logits to f32
    round-off of the different attention chunking (plus the occasional flipped bf16 rounding of a cached k / v),
    over 150 positions (three 64-position chunks per head, several rounds of work items per team)."""
    extra = {"mha-hd64": {}, "gqa-hd64": dict(n_heads=4, n_kv_heads=1), "hd128": dict(hidden=512, n_heads=4, n_kv_heads=2, ffn=1024)}[shape]
    forced = np.random.Generator(np.random.PCG64(17)).integers(0, 512, 150)
    outs = []
    for persistent in (False, True):
        eng = llama.LlamaEngine(llama.preset("tiny", max_seq=160, forward_mode="separate", persistent_forward=persistent, **extra), init="host")
        assert eng.use_fw_persistent == persistent and eng.cfg.head_dim == (128 if shape == "hd128" else 64)
        eng.reset(forced=forced)
        logits = []
        for step in range(150):
            eng.decode_step(graph=(step % 2 == 1))      # eager and replayed steps alternate
            logits.append(eng.logits.cpu().numpy().copy())
        eng.check()
        outs.append((eng.tokens(), np.stack(logits), [k.clone() for k in eng.k_cache], [v.clone() for v in eng.v_cache]))
    (ta, la, ka, va), (tb, lb, kb, vb) = outs
    scale = np.max(np.abs(la))
    assert np.max(np.abs(la - lb)) <= 2e-4 * scale
    agree = sum(a == b for a, b in zip(ta, tb))
    assert agree >= len(ta) - 2                          # a near-tie may flip on 1e-4 logits
    for a, b in zip(ka + va, kb + vb):                   # caches: same bf16 values up to a flipped rounding here and there
        assert (a.float() - b.float()).abs().max().item() <= 2.0 ** -6 * a.float().abs().max().item()
        assert (a != b).float().mean().item() < 0.02
    # the adapter-free backbone runs the same launch
    base = llama.LlamaEngine(llama.preset("tiny", max_seq=32, adapters=False, persistent_forward=True, **extra), init="host")
    assert base.use_fw_persistent
    ref = llama.LlamaEngine(llama.preset("tiny", max_seq=32, adapters=False, persistent_forward=False, **extra), init="host")
    assert base.generate([5, 17, 300], 12) == ref.generate([5, 17, 300], 12)


def test_chained_plain_forward_equals_per_projection_launches(llama):
    """af_gemv_chain (one persistent launch per layer) against one af_gemv_fused launch per projection:
    same tokens, logits equal to f32 summation-order round-off; adapter-free and separate schedules."""
    forced = np.random.Generator(np.random.PCG64(31)).integers(0, 512, 16)
    for kw in (dict(adapters=False), dict(forward_mode="separate")):
        outs = []
        for chain in (True, False):
            eng = llama.LlamaEngine(llama.preset("tiny", max_seq=24, gemv_chain=chain, **kw), init="host")
            assert eng.use_gemv_chain == chain
            eng.reset(forced=forced)
            lg = []
            for _ in range(16):
                eng.decode_step()
                lg.append(eng.logits.cpu().numpy().copy())
            outs.append((eng.tokens(), np.stack(lg)))
        np.testing.assert_allclose(outs[0][1], outs[1][1], rtol=0, atol=1e-4 * np.max(np.abs(outs[1][1])))
        assert outs[0][0] == outs[1][0]


def test_generate_and_base_engine(llama):
    cfg = llama.preset("tiny", max_seq=64)
    eng = llama.LlamaEngine(cfg, init="host")
    toks = eng.generate([5, 17, 300], 12)
    assert len(toks) == 12 and all(0 <= t < cfg.vocab for t in toks)
    assert toks == eng.generate([5, 17, 300], 12, use_graph=False)      # deterministic, graph == eager
    assert eng.max_backbone_deviation() < 0.02
    base = llama.LlamaEngine(llama.preset("tiny", max_seq=64, adapters=False), init="host")
    bt = base.generate([5, 17, 300], 12)
    assert len(bt) == 12
    with pytest.raises(Exception):
        base.fused_switch(None, None)
    with pytest.raises(ValueError):
        llama.preset("tiny", n_kv_heads=3)


def test_tp_shards_are_slices_of_the_full_switch(llama):
    """a rank's switch over its shard equals the same slice of the unsharded
    switch bit for bit (each element's arithmetic is independent of the sharding)."""
    full_cfg = llama.preset("tiny", max_seq=8, compute="fma")
    full = llama.LlamaEngine(full_cfg, init="host")
    dec_a = full.cur.__class__.from_host(llama.GateDecision((1, 6), (0.75, 0.25)))
    dec_b = full.cur.__class__.from_host(llama.GateDecision((6, 3), (0.5, 0.5)))
    full.merge(dec_a)
    full.fused_switch(dec_a, dec_b)
    for rank in range(2):
        cfg = llama.preset("tiny", max_seq=8, compute="fma", tp_size=2, tp_rank=rank)
        one = llama.LlamaEngine(cfg, init="host", comm=llama.NoPeers())   # one shard, no peers: table only
        one.merge(dec_a)
        one.fused_switch(dec_a, dec_b)
        shp = cfg.segment_shapes()
        for li in range(cfg.layers):
            for j, name in enumerate(llama.SEGMENT_NAMES):
                i = li * 7 + j
                fw = full.targets[i].data
                if name in ("q", "k", "v", "gate", "up"):
                    n = shp[name][0]
                    want = fw[rank * n:(rank + 1) * n]
                else:
                    n = shp[name][1]
                    want = fw[:, rank * n:(rank + 1) * n]
                assert torch.equal(one.targets[i].data, want), f"rank {rank} layer {li} {name}"


@pytest.mark.parametrize("shape", ["r8", "r16-gqa", "base"])
def test_batched_unmerged_prefill(llama, shape):
    """SURVEY.md 8f-4 (model.py:408-425, PAPER Eq. 2): the whole prompt in one unmerged batched pass
    == the per-token merged path of the oracle (each token with its own pre-gated decision switched
    into the weights), up to the bf16 rounding of the merged weights; the backbone is not touched;
    KV cache, position and the emitted token are those of the step-by-step path."""
    extra = {"r8": {}, "r16-gqa": dict(experts=16, rank=16, n_heads=4, n_kv_heads=1), "base": dict(adapters=False)}[shape]
    cfg = llama.preset("tiny", max_seq=48, **extra)
    eng = llama.LlamaEngine(cfg, init="host")
    prompt = [int(t) for t in np.random.Generator(np.random.PCG64(21)).integers(0, cfg.vocab, 13)]
    w_before = [_bits(t.data) for t in eng.targets]
    nxt = eng.prefill(prompt)
    assert int(eng.pos_dev.item()) == len(prompt) and eng.steps_done() == len(prompt) and not eng.have_prev
    for before, t in zip(w_before, eng.targets):
        np.testing.assert_array_equal(before, _bits(t.data))            # unmerged: never an sgmm
    got_hidden = eng.last_prefill_hidden.cpu().numpy()
    got_logits = eng.logits.cpu().numpy()
    got_k = [c[:, : len(prompt)].float().cpu().numpy() for c in eng.k_cache]
    got_v = [c[:, : len(prompt)].float().cpu().numpy() for c in eng.v_cache]
    # oracle: merged path, token by token, from pristine weights each time (no drift on its side)
    ora = _oracle_for(eng, llama)
    pristine = [{n: ora.w["layers"][li][n]["bits"].copy() for n in llama.SEGMENT_NAMES} for li in range(cfg.layers)]
    for tkn in prompt:
        if cfg.adapters:
            ora.switch(ora.route(tkn), from_pristine=True, pristine=pristine)
        o_next, o_logits, o_hidden = ora.forward(tkn)
    scale = np.max(np.abs(o_hidden))
    assert np.max(np.abs(got_hidden - o_hidden)) <= 2e-2 * scale
    assert np.max(np.abs(got_logits - o_logits)) <= 2e-2 * np.max(np.abs(o_logits))
    for li in range(cfg.layers):
        np.testing.assert_allclose(got_k[li], ora.kc[li][:, : len(prompt)], atol=3e-2 * max(1.0, np.abs(ora.kc[li]).max()))
        np.testing.assert_allclose(got_v[li], ora.vc[li][:, : len(prompt)], atol=3e-2 * max(1.0, np.abs(ora.vc[li]).max()))
    top2 = np.sort(o_logits)[-2:]
    if top2[1] - top2[0] > 4e-2 * np.max(np.abs(o_logits)):
        assert nxt == o_next
    # the engine's own step-by-step prompt path agrees, and decoding continues from the prefilled cache
    step = llama.LlamaEngine(cfg, init="host")
    step.reset(prompt[0])
    for t in prompt:
        s_nxt = step.decode_step(t)
    np.testing.assert_allclose(step.logits.cpu().numpy(), got_logits, atol=2e-2 * np.max(np.abs(got_logits)))
    a = eng.generate(prompt, 6, prefill="batched")
    b = eng.generate(prompt, 6, prefill="stepwise")
    c = eng.generate(prompt, 6, prefill="batched", use_graph=False)
    assert len(a) == len(b) == 6 and a == c                                # graph == eager after a batched prefill
    assert a[0] == nxt and (a[0] == b[0] or top2[1] - top2[0] <= 4e-2 * np.max(np.abs(o_logits)))
    if cfg.adapters:
        assert eng.max_backbone_deviation() < 0.02
    with pytest.raises(Exception):
        eng.prefill([])
    with pytest.raises(Exception):
        eng.prefill([cfg.vocab])
    with pytest.raises(Exception):
        eng.prefill(list(range(cfg.max_seq + 1)))


class _Lockstep:
    """Exchange layer of `tp` shard engines driven by `tp` threads on ONE GPU: the collectives of
    llama.Collectives, done through shared slots and a barrier (all work is on one stream, so
    enqueue order is execution order).  Exercises the TP forward path without a second device."""

    def __init__(self, tp):
        import threading

        self.tp = tp
        self.slots = [None] * tp
        self.barrier = threading.Barrier(tp, timeout=120)

    def comm(self, llama, rank):
        shared = self

        class Comm(llama.Collectives):
            def __init__(self):
                self.group, self.tp_size = None, shared.tp

            def all_reduce_sum(self, t):
                shared.slots[rank] = t
                shared.barrier.wait()
                total = torch.stack(list(shared.slots)).sum(dim=0)
                shared.barrier.wait()          # every rank has read the originals
                t.copy_(total)
                shared.barrier.wait()

            def broadcast_decision(self, buf):
                shared.slots[rank] = buf
                shared.barrier.wait()
                if rank != 0:
                    buf.copy_(shared.slots[0])
                shared.barrier.wait()

            def argmax_pairs(self, val, idx, out_idx):
                shared.slots[rank] = (val.clone(), idx.clone())
                shared.barrier.wait()
                vals = torch.cat([v.view(1) for v, _ in shared.slots])
                idxs = torch.cat([i.view(1) for _, i in shared.slots])
                best = vals.max()
                winner = torch.where(vals == best, idxs, torch.full_like(idxs, 2 ** 30)).min()
                shared.barrier.wait()
                out_idx.copy_(winner.to(torch.int32).view(1))
                shared.barrier.wait()

        return Comm()


def _run_lockstep(llama, tp, make_cfg, forced, n_steps):
    import threading

    shared = _Lockstep(tp)
    engines = [llama.LlamaEngine(make_cfg(rank), init="host", comm=shared.comm(llama, rank)) for rank in range(tp)]
    tokens, logits, errors = [[] for _ in range(tp)], [[] for _ in range(tp)], []

    def drive(rank):
        try:
            eng = engines[rank]
            eng.reset(forced=forced)
            for _ in range(n_steps):
                tokens[rank].append(eng.decode_step())
                logits[rank].append(eng.logits.clone())
            eng.finalize()
        except BaseException as exc:  # noqa: BLE001 - reported by the main thread
            errors.append((rank, repr(exc)))
            shared.barrier.abort()

    threads = [threading.Thread(target=drive, args=(rank,)) for rank in range(tp)]
    for th in threads:
        th.start()
    for th in threads:
        th.join(timeout=300)
    assert not errors, errors
    return engines, tokens, logits


@pytest.mark.parametrize("forward_mode", ["separate", "chase"])
@pytest.mark.parametrize("tp", [2, 4])
def test_tp_forward_in_lockstep_equals_the_full_model(llama, tp, forward_mode):
    """tp shard engines (column-parallel q/k/v/gate/up, row-parallel o/down, vocab-parallel
    lm_head; decision broadcast, two all-reduces per layer, argmax over (value, index) pairs) decode
    the tokens of the unsharded engine, with the same logits up to the summation order.  "chase": the
    fused switch + GEMV launches per projection, the row-parallel ones followed by an all-reduce of
    their int64 fixed-point accumulators."""
    forced = np.random.Generator(np.random.PCG64(31)).integers(0, 512, 8)
    base = dict(max_seq=16, n_heads=4, n_kv_heads=4)
    full = llama.LlamaEngine(llama.preset("tiny", forward_mode="separate", **base), init="host")
    full.reset(forced=forced)
    want_tokens, want_logits = [], []
    for _ in range(len(forced)):
        want_tokens.append(full.decode_step())
        want_logits.append(full.logits.clone())
    engines, tokens, logits = _run_lockstep(
        llama, tp, lambda r: llama.preset("tiny", tp_size=tp, tp_rank=r, forward_mode=forward_mode, **base), forced, len(forced))
    tol = 2e-3 if forward_mode == "separate" else 4e-3     # chase: x split into bf16 hi + lo, fixed-point sums
    for rank in range(tp):
        assert engines[rank].chase == (forward_mode == "chase") and not getattr(engines[rank], "chase_chained", False)
        assert tokens[rank] == tokens[0], f"rank {rank}"                 # the ranks agree with each other exactly
        assert engines[rank].max_backbone_deviation() < 0.02
    for step in range(len(forced)):
        got = torch.cat([logits[r][step] for r in range(tp)])
        scale = want_logits[step].abs().max().item()
        assert (got - want_logits[step]).abs().max().item() <= tol * scale, f"step {step}"
        top2 = torch.topk(want_logits[step], 2).values
        if (top2[0] - top2[1]).item() > 4 * tol * scale:
            assert tokens[0][step] == want_tokens[step], f"step {step}"


@pytest.mark.parametrize("forward_mode", ["separate", "chase"])
@pytest.mark.parametrize("switch_mode", ["inplace", "from_pristine"])
def test_switch_in_passes_for_more_than_64_stacked_ranks(llama, switch_mode, forward_mode):
    """The fallback for tables whose stacked rank exceeds what ONE launch takes (rank-64 tables: 64; every
    BASELINE configuration fits one K-chunked tcgen05 launch and never gets here): the engine cuts the switch
    into tensor-path passes.  Rank 64, top-2 -- 256 stacked ranks in a steady switch, one expert per pass.
    Against the single CUDA-core pass over all ranks the weights differ by at most one bf16 rounding per
    pass, the logits agree, the backbone is restored."""
    from paper_2603_11873_b200 import _capi

    base = dict(max_seq=16, experts=8, rank=64, top_k=2, switch_mode=switch_mode, refresh_every=0)
    forced = np.random.Generator(np.random.PCG64(41)).integers(0, 512, 6)
    one = llama.LlamaEngine(llama.preset("tiny", split_switch=False, forward_mode="separate", **base), init="host")
    many = llama.LlamaEngine(llama.preset("tiny", forward_mode=forward_mode, **base), init="host")
    # "chase": the last merge pass of every token is fused with the forward (W read once less)
    assert many.split_switch and not one.split_switch and many.chase == (forward_mode == "chase") and not one.chase
    one.reset(forced=forced)
    many.reset(forced=forced)
    n_pass = 8 if switch_mode == "inplace" else 2
    for step in range(len(forced)):
        before = _capi.launch_count()
        a = one.decode_step(graph=False)        # eager: the launches are counted
        single = _capi.launch_count() - before
        before = _capi.launch_count()
        b = many.decode_step(graph=False)
        launches = _capi.launch_count() - before
        assert many.decision() == one.decision()
        want_passes = (2 if switch_mode == "from_pristine" else (4 if step else 2))    # 1 expert of rank 64 per pass
        if forward_mode == "separate":
            assert launches - single == want_passes - 1, f"step {step}: {launches} launches against {single}"
        for i, (ta, tb) in enumerate(zip(one.targets, many.targets)):
            # every pass rounds at the magnitude the element has at that moment: bound the difference by
            # half a bf16 ulp of the matrix's largest element per pass (+ the single pass's own rounding)
            fa, fb = ta.data.float(), tb.data.float()
            ulp = 2.0 ** (np.floor(np.log2(max(fa.abs().max().item(), fb.abs().max().item()))) - 7)
            worst = (fa - fb).abs().max().item() / ulp
            # in place, both engines carry their own roundings from token to token (the drift refresh_every bounds)
            tokens_of_drift = step + 1 if switch_mode == "inplace" else 1
            assert worst <= 0.5 * (n_pass + 1) * tokens_of_drift, f"step {step} segment {i}: {worst} ulp of the largest element"
        scale = one.logits.abs().max().item()
        assert (one.logits - many.logits).abs().max().item() <= 2e-2 * scale
    one.finalize()
    many.finalize()
    assert many.max_backbone_deviation() < 0.05 and one.max_backbone_deviation() < 0.05



@pytest.mark.parametrize("forward_mode", ["separate", "chase", "push"])
def test_tp_two_processes_over_torch_distributed(llama, forward_mode, tmp_path):
    """The lockstep test above with real processes and the engine's own exchange layer: two ranks launched
    by torch.distributed.run, `llama.Collectives` over a gloo group (both ranks on cuda:0 — one GPU here;
    NCCL carries the same calls on a multi-GPU box), decode the unsharded engine's tokens.  "push": the chase schedule with
    `tp_push` -- no all-reduce inside the layers; each rank's chained launches add their partial sums into the other
    PROCESS's accumulators through CUDA IPC mappings and wait on cross-process phase counters (two contexts time-slicing
    one GPU: slow, but the real cross-process path -- handles, offsets, system-scope atomics, the token barrier)."""
    import os
    import socket
    import subprocess
    import sys

    tp = 2
    forced = np.random.Generator(np.random.PCG64(31)).integers(0, 512, 8)
    full = llama.LlamaEngine(llama.preset("tiny", forward_mode="separate", max_seq=16, n_heads=4, n_kv_heads=4), init="host")
    full.reset(forced=forced)
    want_tokens, want_logits = [], []
    for _ in range(len(forced)):
        want_tokens.append(int(full.decode_step()))
        want_logits.append(full.logits.float().cpu().numpy().copy())
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_tp_worker.py")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={tp}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), worker, str(tmp_path), forward_mode],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    ranks = [np.load(tmp_path / f"rank{k}.npz") for k in range(tp)]
    tol = 2e-3 if forward_mode == "separate" else 4e-3
    for k in range(tp):
        assert ranks[k]["tokens"].tolist() == ranks[0]["tokens"].tolist(), f"rank {k}"
        assert float(ranks[k]["deviation"]) < 0.02
    for step in range(len(forced)):
        got = np.concatenate([ranks[k]["logits"][step] for k in range(tp)])
        scale = np.abs(want_logits[step]).max()
        assert np.abs(got - want_logits[step]).max() <= tol * scale, f"step {step}"
        top2 = np.sort(want_logits[step])[-2:]
        if top2[1] - top2[0] > 4 * tol * scale:
            assert int(ranks[0]["tokens"][step]) == want_tokens[step], f"step {step}"


@pytest.mark.parametrize("forward_mode", ["separate", "chase"])
def test_tp_step_with_nccl_collectives_captures(forward_mode):
    """A TP shard's step — the engine's collectives on torch's NCCL process group — captured as a CUDA graph
    (opt-in, AF_TP_GRAPH=1) replays to the eager step's tokens and weights.  One-rank NCCL group (one GPU
    here): the capture mechanics, not the exchange, are what this covers."""
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_tp_graph_worker.py")
    r = subprocess.run([sys.executable, worker, forward_mode, str(port)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "TP_GRAPH_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
