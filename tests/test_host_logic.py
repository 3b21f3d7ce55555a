"""Host-side logic that needs no GPU: validation order and error classes of the mirrored
reference API, dispatch accounting, Llama shard algebra and byte formulas, and the N>1 exchange
layer on a world_size-2 gloo group."""

import os
import socket

import numpy as np
import pytest
import torch

import paper_2603_11873_b200 as af
from paper_2603_11873_b200 import llama
from paper_2603_11873_b200.routing import decision_to_struct


# ------------------------------------------------------------------ reference API ----


def test_model_config_validation():
    # /root/reference/pkg/src/lorafuse/model.py:101-119
    af.ModelConfig().validate()
    for bad in (dict(layers=0), dict(vocab=1), dict(top_k=9, experts=8), dict(rank=65, hidden=64), dict(precision="double"),
                dict(strategy="pre_gated_fused"), dict(refresh_every=-2), dict(seed=1.5), dict(hidden=True),
                dict(compute="fast"), dict(switch_mode="copy")):
        with pytest.raises(ValueError):
            af.ModelConfig(**bad).validate()
    cfg = af.ModelConfig.from_dict(af.ModelConfig(strategy=af.Strategy.BASE).to_dict())
    assert cfg.strategy is af.Strategy.BASE
    assert af.Strategy.PRE_GATED_FUSED.merges_backbone and not af.Strategy.PRE_GATED_NAIVE.merges_backbone


def test_recorder_contract():
    # linalg.py:125-159
    rec = af.DispatchRecorder()
    rec.record("gemm", 10, 20, "router")
    mark = rec.mark()
    rec.record("sgmm", 5, 6)
    assert [e.kind for e in rec.events_since(mark)] == ["sgmm"]
    assert rec.counts() == {"gemm": 1, "sgmm": 1, "elementwise": 0, "reduce": 0}
    with pytest.raises(ValueError):
        rec.record("launch", 0, 0)
    with pytest.raises(ValueError):
        rec.record("gemm", -1, 0)
    summary = rec.reset_and_report()
    assert summary.total_flops == 15 and summary.total_bytes == 26 and not rec.events


def test_matrix_and_segment_validation_without_a_device():
    m = af.Matrix(np.zeros((2, 3)), "single", device="cpu")
    assert (m.rows, m.cols, m.itemsize, m.precision) == (2, 3, 4, "single")
    with pytest.raises(af.DimensionError):
        af.Matrix(np.zeros(3), "single", device="cpu")
    with pytest.raises(af.PrecisionError):
        af.Matrix(np.zeros((1, 1)), "half", device="cpu")
    with pytest.raises(af.PrecisionError):
        af.Matrix.zeros(1, 1, "double", device="cpu")
    with pytest.raises(af.DimensionError):
        af.Matrix.zeros(-1, 1, "single", device="cpu")
    with pytest.raises(ValueError):
        af.TileConfig(m=0)
    t = af.Matrix(np.zeros((4, 4)), "single", device="cpu")
    up = af.Matrix(np.zeros((4, 2)), "single", device="cpu")
    dn = af.Matrix(np.zeros((2, 4)), "single", device="cpu")
    af.Segment(dn, up, t).validate()
    af.Segment(dn, up, af.Matrix(np.zeros((4, 4)), "bf16", device="cpu")).validate()  # bf16 target, f32 gated factors
    with pytest.raises(af.DimensionError):
        af.Segment(dn, af.Matrix(np.zeros((4, 3)), "single", device="cpu"), t).validate()
    with pytest.raises(af.DimensionError):
        af.Segment(dn, up, af.Matrix(np.zeros((5, 4)), "single", device="cpu")).validate()
    with pytest.raises(af.PrecisionError):
        af.Segment(af.Matrix(dn.data, "bf16", device="cpu"), up, t).validate()
    with pytest.raises(af.DimensionError):
        af.SegmentTable([]).validate()
    with pytest.raises(af.AliasingError):
        af.SegmentTable([af.Segment(dn, up, t), af.Segment(dn, up, t)]).validate()
    rec = af.DispatchRecorder()
    with pytest.raises(ValueError):
        af.sgmm(af.SegmentTable([af.Segment(dn, up, t)]), 2, rec)
    with pytest.raises(ValueError):
        af.gemm_accumulate_inplace(t, up, dn, 0, rec)
    with pytest.raises(af.DimensionError):
        af.gemm_accumulate_inplace(t, up, af.Matrix(np.zeros((3, 4)), "single", device="cpu"), 1, rec)
    if not torch.cuda.is_available():
        with pytest.raises(af.DeviceError):      # validation passed; the launch itself has no CPU fallback
            af.sgmm(af.SegmentTable([af.Segment(dn, up, t)]), 1, rec)
    assert not rec.events


def test_adapter_algebra_validation():
    # adapters.py:150-162, 199-200, 224-229
    e = af.ConcatAdapter.empty(4, 6, "single", device="cpu")
    e.validate()
    assert (e.s, e.d_in, e.d_out) == (0, 6, 4)
    bad = af.ConcatAdapter(af.Matrix(np.zeros((2, 6)), "single", device="cpu"), af.Matrix(np.zeros((4, 2)), "single", device="cpu"), ())
    with pytest.raises(af.DimensionError):
        bad.validate()
    ex = af.LoraExpert(af.Matrix(np.ones((2, 6)), "single", device="cpu"), af.Matrix(np.ones((4, 2)), "single", device="cpu"))
    ex.validate()
    with pytest.raises(af.DimensionError):
        af.LoraExpert(af.Matrix(np.ones((2, 6)), "single", device="cpu"), af.Matrix(np.ones((4, 3)), "single", device="cpu")).validate()
    with pytest.raises(IndexError):
        af.concat_gated((ex, ex), af.GateDecision((0, 2), (0.5, 0.5)))
    with pytest.raises(ValueError):
        af.concat_gated((ex, ex), af.GateDecision((), ()))
    cat = af.concat_gated((ex, ex), af.GateDecision((1, 0), (0.75, 0.25)))
    assert cat.s == 4 and cat.provenance == ((1, 0.75, 1), (0, 0.25, 1))
    assert np.array_equal(cat.down_cat.numpy()[:2], np.full((2, 6), 0.75, np.float32))     # gate folded into DOWN only
    assert np.array_equal(cat.up_cat.numpy(), np.ones((4, 4), np.float32))
    sw = af.build_switch(cat, cat)
    assert sw.s == 8 and [p[2] for p in sw.provenance] == [-1, -1, 1, 1]
    assert np.array_equal(sw.down_cat.numpy()[:4], -cat.down_cat.numpy())
    assert af.build_switch(e, cat).provenance == cat.provenance                            # empty prev -> cur
    with pytest.raises(af.DimensionError):
        af.build_switch(af.ConcatAdapter.empty(5, 6, "single", device="cpu"), cat)
    with pytest.raises(af.DimensionError):
        af.merge_all([af.Matrix(np.zeros((4, 6)), "single", device="cpu")], [], 1, af.DispatchRecorder())


def test_decision_struct_round_trip():
    d = decision_to_struct(af.GateDecision((5, 2, 7), (0.5, 0.25, 0.25)))
    assert d.k == 3 and list(d.ids)[:3] == [5, 2, 7] and abs(d.weights[1] - 0.25) < 1e-9
    assert decision_to_struct(None) is None
    with pytest.raises(ValueError):
        decision_to_struct(af.GateDecision(tuple(range(9)), tuple([1 / 9] * 9)))


# ------------------------------------------------------------------ Llama shard algebra ----


def test_preset_bytes_match_the_scope_table():
    # W elements and switch bytes of C2 / C3; decode floor bytes
    c2 = llama.preset("llama2-7b")
    assert c2.layers * sum(o * i for o, i in c2.segment_shapes().values()) == 6_476_005_376
    assert c2.switch_bytes() == 26_063_929_344
    c3 = llama.preset("llama3-8b")
    assert c3.layers * sum(o * i for o, i in c3.segment_shapes().values()) == 6_979_321_856
    assert abs(c3.switch_bytes() / 1e9 - 28.253) < 0.01
    c4 = llama.preset("llama2-13b", tp_size=4)
    assert 4 * c4.layers * sum(o * i for o, i in c4.segment_shapes().values()) == 12_687_769_600
    assert llama.preset("llama2-70b", tp_size=8).segment_shapes()["k"] == (128, 8192)   # one kv head per rank
    assert c2.switch_bytes(steady=False) < c2.switch_bytes()
    with pytest.raises(ValueError):
        llama.preset("llama2-70b", tp_size=16)
    with pytest.raises(af.ConfigError):
        llama.preset("llama-9b")


@pytest.mark.parametrize("tp", [2, 4])
def test_shards_tile_the_full_tensors(tp):
    base = dict(layers=1, hidden=64, ffn=128, n_heads=8, n_kv_heads=4, vocab=64, experts=3, rank=8, top_k=2)
    full = llama.host_weights(llama.LlamaConfig(**base))
    shards = [llama.host_weights(llama.LlamaConfig(**base, tp_size=tp, tp_rank=r)) for r in range(tp)]
    for name in llama.SEGMENT_NAMES:
        f = full["layers"][0][name]
        parts = [s["layers"][0][name] for s in shards]
        if name in ("q", "k", "v", "gate", "up"):       # column-parallel: W rows and UP rows split, DOWN replicated
            assert np.array_equal(np.concatenate([p["w"] for p in parts], axis=0), f["w"])
            assert np.array_equal(np.concatenate([p["up"] for p in parts], axis=1), f["up"])
            assert all(np.array_equal(p["down"], f["down"]) for p in parts)
        else:                                            # row-parallel: W cols and DOWN cols split, UP replicated
            assert np.array_equal(np.concatenate([p["w"] for p in parts], axis=1), f["w"])
            assert np.array_equal(np.concatenate([p["down"] for p in parts], axis=2), f["down"])
            assert all(np.array_equal(p["up"], f["up"]) for p in parts)
        # the delta of a shard is the shard of the delta: B_rows A  /  B A_cols
        g = np.float32(0.625)
        delta = f["up"][1] @ (g * f["down"][1])
        for r, p in enumerate(parts):
            d_sh = p["up"][1] @ (g * p["down"][1])
            n0 = d_sh.shape[0] if name in ("q", "k", "v", "gate", "up") else d_sh.shape[1]
            want = delta[r * n0:(r + 1) * n0] if name in ("q", "k", "v", "gate", "up") else delta[:, r * n0:(r + 1) * n0]
            np.testing.assert_allclose(d_sh, want, rtol=1e-6, atol=1e-7)
    assert np.array_equal(np.concatenate([s["lm_head"] for s in shards], axis=0), full["lm_head"])
    cos, sin = llama.rope_tables(llama.LlamaConfig(**base))
    assert cos.shape == (256, 4) and np.allclose(cos[0], 1) and np.allclose(sin[0], 0)


# ------------------------------------------------------------------ world_size-2 gloo ----


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = llama.Collectives(None, world)
        # (1) the switch path's only collective: rank 0's 128-byte decision record
        gate = af.GateDecision((3, 1), (0.75, 0.25)) if rank == 0 else af.GateDecision((0, 0), (0.5, 0.5))
        buf = torch.frombuffer(bytearray(bytes(decision_to_struct(gate))), dtype=torch.uint8).clone()
        comm.broadcast_decision(buf)
        got = af.DeviceDecision(buf=buf).to_host()
        # (2) row-parallel partial sums
        part = torch.full((8,), float(rank + 1))
        comm.all_reduce_sum(part)
        # (3) vocab-parallel argmax: largest value wins, lowest index on ties
        val = torch.tensor([2.5]) if rank == 0 else torch.tensor([2.5])
        idx = torch.tensor([7 + 100 * rank], dtype=torch.int32)
        out = torch.zeros(1, dtype=torch.int32)
        comm.argmax_pairs(val, idx, out)
        val2 = torch.tensor([1.0 + rank])
        out2 = torch.zeros(1, dtype=torch.int32)
        comm.argmax_pairs(val2, idx, out2)
        q.put((rank, got, part.tolist(), int(out.item()), int(out2.item())))
    finally:
        dist.destroy_process_group()


def test_exchange_layer_world_size_2_gloo():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, part, tie_idx, max_idx in results:
        assert got == af.GateDecision((3, 1), (0.75, 0.25))       # every rank switches on rank 0's decision
        assert part == [3.0] * 8
        assert tie_idx == 7                                        # tie -> lowest token id (model.py:396)
        assert max_idx == 107                                      # rank 1 holds the larger value


def test_collectives_need_an_initialised_group():
    with pytest.raises(af.StateError):
        llama.Collectives(None, 2)
    llama.Collectives(None, 1).all_reduce_sum(torch.zeros(1))       # tp=1: no-ops


# ------------------------------------------------------------------ round-2 host logic ----


def test_refresh_period_defaults_and_validation():
    """model.py:344-349 `refresh_every`: the reference's default (never) stays for f32; bf16 storage refreshes every 16
    tokens unless told otherwise; -1 turns it off."""
    assert af.ModelConfig(precision="single").effective_refresh_every == 0
    assert af.ModelConfig(precision="bf16").effective_refresh_every == 16
    assert af.ModelConfig(precision="bf16", refresh_every=5).effective_refresh_every == 5
    assert af.ModelConfig(precision="bf16", refresh_every=-1).effective_refresh_every == 0
    assert af.ModelConfig(precision="bf16", switch_mode="from_pristine").effective_refresh_every == 0
    assert af.ModelConfig(precision="bf16", strategy=af.Strategy.BASE).effective_refresh_every == 0
    with pytest.raises(ValueError):
        af.ModelConfig(refresh_every=-2).validate()
    assert llama.preset("tiny").refresh_every == 16
    with pytest.raises(ValueError):
        llama.preset("tiny", refresh_every=-1)
    with pytest.raises(ValueError):
        llama.preset("tiny", refresh_every=True)


def test_status_word_messages_and_exception_classes():
    """af_flag_message / _capi.raise_for_flag: what a kernel raised on the device maps onto the reference's classes."""
    from paper_2603_11873_b200 import _capi, errors

    L = _capi.lib()
    assert b"outside the bank" in L.af_flag_message(_capi.AF_EINDEX)
    assert b"phase barrier" in L.af_flag_message(_capi.AF_ECUDA)
    _capi.raise_for_flag(0)
    with pytest.raises(IndexError):
        _capi.raise_for_flag(_capi.AF_EINDEX)
    with pytest.raises(ValueError):
        _capi.raise_for_flag(_capi.AF_EVALUE)
    with pytest.raises(errors.StateError):
        _capi.raise_for_flag(_capi.AF_ESTATE)
    with pytest.raises(errors.DeviceError):
        _capi.raise_for_flag(_capi.AF_ECUDA)


def test_forward_phase_table_validation():
    """af_forward_validate checks the HOST copy of the persistent forward's phase table before it is uploaded
    (no device needed): shapes, alignment, prologue / epilogue operands, phase order."""
    import ctypes

    from paper_2603_11873_b200 import _capi, errors

    L = _capi.lib()
    P = _capi.FwPhase
    assert ctypes.sizeof(P) == 88

    def gemv(**kw):
        base = dict(w=0x1000, x=0x2000, out=0x3000, res=None, norm_w=None, k_cache=None, v_cache=None, ld=256, rows=64, cols=256,
                    eps=1e-5, prologue=_capi.AF_PRO_NONE, epilogue=_capi.AF_EPI_NONE, kind=_capi.AF_FW_GEMV)
        base.update(kw)
        return P(**base)

    att_p = P(w=None, x=0x2000, out=None, res=None, norm_w=None, k_cache=0x4000, v_cache=0x5000, ld=0, rows=0, cols=0, eps=0.0,
              prologue=0, epilogue=0, kind=_capi.AF_FW_ATTN_PARTIAL)
    att_c = P(w=None, x=None, out=0x6000, res=None, norm_w=None, k_cache=None, v_cache=None, ld=0, rows=0, cols=0, eps=0.0,
              prologue=0, epilogue=0, kind=_capi.AF_FW_ATTN_COMBINE)

    def check(phases, heads=4, kv=2, hd=64):
        arr = (P * len(phases))(*phases)
        mc = ctypes.c_int32()
        _capi.check(L.af_forward_validate(arr, len(phases), heads, kv, hd, ctypes.byref(mc)))
        return mc.value

    assert check([gemv(), att_p, att_c, gemv(cols=512, ld=512)]) == 512
    with pytest.raises(errors.DimensionError):
        check([gemv()], hd=96)                                      # head_dim 64 or 128
    with pytest.raises(errors.DimensionError):
        check([gemv(cols=250, ld=250)])                             # 16-byte rows
    with pytest.raises(ValueError):
        check([gemv(prologue=_capi.AF_PRO_RMSNORM)])                # RMSNorm without its weight
    with pytest.raises(ValueError):
        check([gemv(epilogue=_capi.AF_EPI_RESIDUAL)])               # residual epilogue without a residual
    with pytest.raises(errors.AliasingError):
        check([gemv(out=0x2000)])
    with pytest.raises(ValueError):
        check([gemv(), att_c])                                      # a combine needs its partials phase in front
    with pytest.raises(ValueError):
        check([gemv(kind=7)])
    with pytest.raises(errors.DimensionError):
        check([gemv()], heads=3, kv=2)


def test_peer_buffer_contract_and_peer_calls_validate_without_a_device():
    """`llama.PeerBuffer` (what a TP rank hands the engine for tp_push) and the argument checks of the peer calls of the
    C ABI, which run before anything touches a device."""
    import ctypes

    from paper_2603_11873_b200 import _capi
    from paper_2603_11873_b200.errors import DimensionError

    buf = llama.PeerBuffer(torch.zeros(16, dtype=torch.int64), [-4096, 0, 4096])
    assert buf.offsets == [-4096, 0, 4096] and buf.tensor.numel() == 16
    with pytest.raises(ValueError):
        llama.PeerBuffer(torch.zeros(16, dtype=torch.int64), [4096, 8192])      # this rank (0) is missing
    with pytest.raises(ValueError):
        llama.PeerBuffer(torch.zeros(16, dtype=torch.int64), [0, 0])
    with pytest.raises(DimensionError):
        llama.PeerBuffer(torch.zeros(16, dtype=torch.int32), [0])
    assert llama.LlamaConfig().tp_push is None
    L = _capi.lib()
    offs = (ctypes.c_int64 * 2)(0, 4096)
    assert L.af_group_set_peers(None, 2, offs, 1) == _capi.AF_EVALUE             # no group
    assert L.af_peer_barrier(None, None, 2, offs, None, None) == _capi.AF_EVALUE
    assert L.af_peer_wait(None, 1, None, None) == _capi.AF_EVALUE
    assert L.af_peer_bcast(None, None, None, 128, 1, None, None, 2, offs, None, None) == _capi.AF_EVALUE
    assert L.af_peer_argmax(None, None, None, 0, None, None, 2, offs, None, None, None) == _capi.AF_EVALUE
