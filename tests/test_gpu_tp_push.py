"""Tensor parallelism without a collective between the launches (include/adafuse_b200.h `af_group_set_peers`,
`af_peer_barrier`, `af_peer_wait`; no reference counterpart -- the reference is single-process and BASELINE
configs[3..4] only name TP 2 / 4 / 8).

One B200 plays both ranks: two shard tables, two streams, two chained launches of 40 CTAs each that are resident
TOGETHER and push the partial sums of their row-parallel phases (o, down) into each other's accumulators -- the
same system-scope atomics and cross-rank phase counters that run over NVLink peer mappings between GPUs; here the
"peer mapping" is a second region of one allocation.

The sums are integers (fixed point, 2^-40), the 128-column strips of a row are the same whether the row lives on
one rank or is split over two, and a merged tile depends on its own rows / columns of the factors only: so the
two-rank result must be BIT-IDENTICAL to the single-rank chain on the unsharded matrices -- accumulators, residual
streams and merged weights."""

import pytest
import torch

pytestmark = pytest.mark.gpu

D, F, N_EXP, RANK = 512, 1280, 6, 8      # a shard's largest phase is 40 tiles: two launches of 40 CTAs are resident together


@pytest.fixture(scope="module")
def af():
    import paper_2603_11873_b200 as af

    return af


def _decision(ids, weights):
    from paper_2603_11873_b200.routing import DeviceDecision, GateDecision

    return DeviceDecision.from_host(GateDecision(tuple(ids), tuple(weights)), torch.device("cuda"))


def _full_model(seed=11):
    """Unsharded matrices and factors of one block: o | gate up | down | q k v (all `d_out x d_in`)."""
    g = torch.Generator(device="cuda").manual_seed(seed)

    def u(shape, fan):
        return (torch.empty(shape, device="cuda").uniform_(-1, 1, generator=g) * fan ** -0.5).to(torch.bfloat16)

    shapes = [(D, D), (F, D), (F, D), (D, F), (D, D), (D, D), (D, D)]
    w = [u((o, i), i) for o, i in shapes]
    down = [u((N_EXP, RANK, i), i) for o, i in shapes]      # A: rank x d_in
    up = [u((N_EXP, o, RANK), RANK) for o, i in shapes]      # B: d_out x rank
    return shapes, w, down, up


def _shard(w, down, up, rank, tp):
    """Row-parallel (split d_in: o, down) and column-parallel (split d_out: gate, up, q, k, v) shards of rank `rank`."""
    row_parallel = [True, False, False, True, False, False, False]
    ws, dns, ups = [], [], []
    for i, rp in enumerate(row_parallel):
        if rp:
            n = w[i].shape[1] // tp
            sl = slice(rank * n, (rank + 1) * n)
            ws.append(w[i][:, sl].contiguous())
            dns.append(down[i][:, :, sl].contiguous())
            ups.append(up[i].clone())
        else:
            n = w[i].shape[0] // tp
            sl = slice(rank * n, (rank + 1) * n)
            ws.append(w[i][sl].contiguous())
            dns.append(down[i].clone())
            ups.append(up[i][:, sl].contiguous())
    return ws, dns, ups


def _table(ws, dns, ups):
    from paper_2603_11873_b200.adapters import SwitchTable
    from paper_2603_11873_b200.linalg import Matrix

    targets = [Matrix(t.clone(), "bf16") for t in ws]
    return targets, SwitchTable(targets, [t.clone() for t in dns], [t.clone() for t in ups])


PHASE_IDS = [[0], [1, 2], [3], [4, 5, 6]]


def _inputs():
    g = torch.Generator(device="cuda").manual_seed(2)
    attn = torch.empty(D, device="cuda").uniform_(-1, 1, generator=g)
    xa = torch.empty(D, device="cuda").uniform_(-1, 1, generator=g)
    nw1 = 1.0 + 0.1 * torch.empty(D, device="cuda").uniform_(-1, 1, generator=g)
    nw2 = 1.0 + 0.1 * torch.empty(D, device="cuda").uniform_(-1, 1, generator=g)
    return attn, xa, nw1, nw2


def _phases(acc, attn_in, xa, xb, xa2, nw1, nw2):
    return [dict(acc_out=acc[0], xin=attn_in),
            dict(acc_out=acc[1], acc_in=acc[0], res=xa, h_out=xb, prologue="rmsnorm", norm_w=nw1, eps=1e-5),
            dict(acc_out=acc[2], acc_in=acc[1], prologue="silu_mul"),
            dict(acc_out=acc[3], acc_in=acc[2], res=xb, h_out=xa2, prologue="rmsnorm", norm_w=nw2, eps=1e-5)]


def test_two_ranks_on_one_gpu_equal_the_single_rank_chain(af):
    from paper_2603_11873_b200.adapters import SegmentGroup

    tp = 2
    shapes, w, down, up = _full_model()
    prev, cur = _decision((1, 4), (0.7, 0.3)), _decision((4, 2), (0.55, 0.45))
    attn, xa, nw1, nw2 = _inputs()

    # ---- single rank, unsharded ----
    tg, tab = _table(w, down, up)
    tab.switch(None, prev, max_k=2)
    xb, xa2 = torch.zeros(D, device="cuda"), torch.zeros(D, device="cuda")
    acc = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (D, 2 * F, D, 3 * D)]
    done = torch.zeros(4, dtype=torch.int32, device="cuda")
    grp = SegmentGroup(tab, PHASE_IDS)
    grp.switch_gemv_chain(prev, cur, _phases(acc, attn, xa, xb, xa2, nw1, nw2), done, max_k=2)
    tab.status()
    want = dict(acc=[a.clone() for a in acc], xb=xb.clone(), xa2=xa2.clone(), w=[t.data.clone() for t in tg])

    # ---- two ranks: one buffer, one region per rank, holding what the peers write: o and down sums + the counters ----
    region = 2 * D + 16                                  # int64 words: acc o | acc down | 4 int32 counters (+ pad)
    shared = torch.zeros(tp * region, dtype=torch.int64, device="cuda")
    ranks = []
    for r in range(tp):
        ws, dns, ups = _shard(w, down, up, r, tp)
        tg_r, tab_r = _table(ws, dns, ups)
        assert tab_r.info()["umma_path"]
        tab_r.switch(None, prev, max_k=2)
        reg = shared[r * region: (r + 1) * region]
        acc_r = [reg[:D], torch.zeros(2 * F // tp, dtype=torch.int64, device="cuda"), reg[D: 2 * D],
                 torch.zeros(3 * D // tp, dtype=torch.int64, device="cuda")]
        done_r = reg[2 * D: 2 * D + 2].view(torch.int32)
        grp_r = SegmentGroup(tab_r, PHASE_IDS)
        assert 2 * grp_r.grid <= 148
        offs = [(q - r) * region * 8 for q in range(tp)]
        grp_r.set_peers(offs, reduce_phases=[0, 2])
        n_local = D // tp                                 # this rank's heads: its slice of the attention output
        ranks.append(dict(tg=tg_r, tab=tab_r, grp=grp_r, acc=acc_r, done=done_r, xb=torch.zeros(D, device="cuda"),
                          xa2=torch.zeros(D, device="cuda"), attn=attn[r * n_local: (r + 1) * n_local].contiguous(),
                          stream=torch.cuda.Stream()))
    torch.cuda.synchronize()
    for rk in ranks:                                      # both launches in flight together, neither can finish alone
        with torch.cuda.stream(rk["stream"]):
            rk["grp"].switch_gemv_chain(prev, cur, _phases(rk["acc"], rk["attn"], xa, rk["xb"], rk["xa2"], nw1, nw2), rk["done"], max_k=2)
    torch.cuda.synchronize()
    for r, rk in enumerate(ranks):
        rk["tab"].status()
        # counters: a reduced phase is reported by the CTAs of both ranks, a local one by this rank's
        n_cta = rk["grp"].grid
        assert rk["done"][:3].tolist() == [tp * n_cta, n_cta, tp * n_cta]
        assert torch.equal(rk["acc"][0], want["acc"][0]) and torch.equal(rk["acc"][2], want["acc"][2])      # all-reduced sums
        f_loc, d_loc = F // tp, D // tp
        gate_up = torch.cat([want["acc"][1][r * f_loc: (r + 1) * f_loc], want["acc"][1][F + r * f_loc: F + (r + 1) * f_loc]])
        assert torch.equal(rk["acc"][1], gate_up)
        qkv = torch.cat([want["acc"][3][m * D + r * d_loc: m * D + (r + 1) * d_loc] for m in range(3)])
        assert torch.equal(rk["acc"][3], qkv)
        assert torch.equal(rk["xb"], want["xb"]) and torch.equal(rk["xa2"], want["xa2"])                    # residual streams
        ws, _, _ = _shard(want["w"], down, up, r, tp)                                                        # merged weights
        for got, ref in zip(rk["tg"], ws):
            assert torch.equal(got.data, ref)
    assert float(want["acc"][3].abs().max()) > 0


def test_last_phase_reduced_needs_its_own_counter_and_wait(af):
    """A chain that ENDS in a row-parallel phase (the last layer: o -> gate|up -> down) reports that phase too; the
    consumer is a later launch, ordered behind `peer_wait` on the extra counter."""
    from paper_2603_11873_b200.adapters import SegmentGroup, peer_wait
    from paper_2603_11873_b200.errors import DimensionError

    tp = 2
    shapes, w, down, up = _full_model(seed=12)
    prev, cur = _decision((0, 3), (0.6, 0.4)), _decision((3, 5), (0.5, 0.5))
    attn, xa, nw1, _ = _inputs()
    ids = PHASE_IDS[:3]

    tg, tab = _table(w, down, up)
    tab.switch(None, prev, max_k=2)
    xb = torch.zeros(D, device="cuda")
    acc = [torch.zeros(n, dtype=torch.int64, device="cuda") for n in (D, 2 * F, D)]
    done = torch.zeros(4, dtype=torch.int32, device="cuda")
    SegmentGroup(tab, ids).switch_gemv_chain(
        prev, cur, _phases(acc + [None], attn, xa, xb, None, nw1, None)[:3], done, max_k=2)
    tab.status()

    region = 2 * D + 16
    shared = torch.zeros(tp * region, dtype=torch.int64, device="cuda")
    ranks = []
    for r in range(tp):
        ws, dns, ups = _shard(w, down, up, r, tp)
        tg_r, tab_r = _table(ws, dns, ups)
        tab_r.switch(None, prev, max_k=2)
        reg = shared[r * region: (r + 1) * region]
        acc_r = [reg[:D], torch.zeros(2 * F // tp, dtype=torch.int64, device="cuda"), reg[D: 2 * D]]
        done_r = reg[2 * D: 2 * D + 2].view(torch.int32)
        grp_r = SegmentGroup(tab_r, ids)
        grp_r.set_peers([(q - r) * region * 8 for q in range(tp)], reduce_phases=[0, 2])
        with pytest.raises(DimensionError):              # three counters now: two boundaries + the reduced last phase
            grp_r.switch_gemv_chain(prev, cur, _phases(acc_r + [None], attn[:D // tp].contiguous(), xa, xb, None, nw1, None)[:3],
                                    torch.zeros(2, dtype=torch.int32, device="cuda"), max_k=2)
        n_local = D // tp
        ranks.append(dict(tab=tab_r, grp=grp_r, acc=acc_r, done=done_r, xb=torch.zeros(D, device="cuda"),
                          attn=attn[r * n_local: (r + 1) * n_local].contiguous(), stream=torch.cuda.Stream(),
                          out=torch.zeros(D, dtype=torch.int64, device="cuda")))
    torch.cuda.synchronize()
    # (one GPU plays both ranks: launches that wait for each other are enqueued back to back, so that even if the two
    #  streams share a hardware queue nothing a launch waits for sits behind one of its own successors)
    for rk in ranks:
        with torch.cuda.stream(rk["stream"]):
            rk["grp"].switch_gemv_chain(prev, cur, _phases(rk["acc"] + [None], rk["attn"], xa, rk["xb"], None, nw1, None)[:3], rk["done"], max_k=2)
    for rk in ranks:
        with torch.cuda.stream(rk["stream"]):
            peer_wait(rk["done"][2:3], tp * rk["grp"].grid)        # ... then the consumer of the reduced sums, on the same stream
            rk["out"].copy_(rk["acc"][2])
    torch.cuda.synchronize()
    for rk in ranks:
        rk["tab"].status()
        n_cta = rk["grp"].grid
        assert rk["done"][:3].tolist() == [tp * n_cta, n_cta, tp * n_cta]
        assert torch.equal(rk["out"], acc[2])


def test_peer_barrier_between_two_streams(af):
    """`af_peer_barrier`: a monotonic counter every rank bumps on every rank; round k completes when the own counter
    has reached k * n_peers.  Two streams play the ranks, several rounds (the time-out of a rank left alone:
    test_a_missing_peer_times_out_and_later_waits_fail_fast)."""
    from paper_2603_11873_b200.adapters import peer_barrier

    tp = 2
    shared = torch.zeros(tp * 4, dtype=torch.int32, device="cuda")         # one 16-byte region per rank
    epochs = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(tp)]
    streams = [torch.cuda.Stream() for _ in range(tp)]
    marks = torch.zeros(tp, 3, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for rnd in range(3):
        for r in range(tp):                                   # (the two barriers of a round back to back, see above)
            with torch.cuda.stream(streams[r]):
                peer_barrier(shared[r * 4: r * 4 + 1], epochs[r], [(q - r) * 16 for q in range(tp)])
        for r in range(tp):
            with torch.cuda.stream(streams[r]):
                marks[r, rnd] = rnd + 1
    torch.cuda.synchronize()
    assert shared[0].item() == 3 * tp and shared[4].item() == 3 * tp
    assert [e.item() for e in epochs] == [3, 3] and marks.tolist() == [[1, 2, 3]] * tp


def test_set_peers_validation(af):
    from paper_2603_11873_b200.adapters import SegmentGroup
    from paper_2603_11873_b200.errors import AliasingError, DimensionError

    shapes, w, down, up = _full_model(seed=13)
    tg, tab = _table(w, down, up)
    grp = SegmentGroup(tab, PHASE_IDS)
    with pytest.raises(ValueError):
        grp.set_peers([0, 4096], reduce_phases=[4])          # the chain has phases 0..3
    with pytest.raises(ValueError):
        grp.set_peers([8, 4096], reduce_phases=[0])          # this rank (offset 0) is missing
    with pytest.raises(AliasingError):
        grp.set_peers([0, 4096, 4096], reduce_phases=[0])
    with pytest.raises(DimensionError):
        grp.set_peers([0, 4100], reduce_phases=[0])          # accumulators are 8-byte words
    with pytest.raises(ValueError):
        grp.set_peers([0] + [4096 * i for i in range(1, 9)], reduce_phases=[0])   # at most 8 ranks
    grp.set_peers([0, 4096], reduce_phases=[0, 2])
    grp.set_peers([], reduce_phases=[])                        # cleared: a single rank again
    assert grp.n_peers == 0


def test_engine_with_push_enabled_equals_the_plain_engine(af):
    """`LlamaConfig.tp_push=True` on ONE rank (the only peer is the rank itself): the engine runs the TP-push step --
    accumulators and counters in the peer buffer, the token barrier, o and down pushed with system-scope atomics, the
    wait for the last layer's down projection -- and must reproduce the plain engine bit for bit: tokens, logits and
    the weights the switches leave behind."""
    import numpy as np

    from paper_2603_11873_b200 import llama

    forced = np.random.Generator(np.random.PCG64(5)).integers(0, 512, 12)
    outs = []
    for push in (False, True):
        cfg = llama.preset("tiny", max_seq=32, forward_mode="chase", tp_push=push)
        eng = llama.LlamaEngine(cfg, init="host")
        assert eng.chase and eng.chase_chained and eng.tp_push == push
        if push:
            assert eng.peer_buf.offsets == [0] and eng.groups[0]["mid"].n_peers == 1
        eng.reset(forced=forced)
        toks, logits = [], []
        for _ in forced:
            toks.append(eng.decode_step(graph=False))
            logits.append(eng.logits.clone())
        eng.check()
        if push:
            assert int(eng.peer_epoch.item()) == len(forced) and int(eng.peer_counter.item()) == len(forced)
        outs.append((toks, logits, [t.data.clone() for t in eng.targets]))
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert torch.equal(a, b)
    for a, b in zip(outs[0][2], outs[1][2]):
        assert torch.equal(a, b)


def test_engine_push_step_replays_as_a_graph(af):
    """The push step has no library collective inside the layers: it captures and replays like the single-rank step
    (the barrier's epoch lives on the device)."""
    import numpy as np

    from paper_2603_11873_b200 import llama

    forced = np.random.Generator(np.random.PCG64(6)).integers(0, 512, 10)
    runs = []
    for graph in (False, True):
        eng = llama.LlamaEngine(llama.preset("tiny", max_seq=32, forward_mode="chase", tp_push=True), init="host")
        eng.reset(forced=forced)
        runs.append([eng.decode_step(graph=graph) for _ in forced])
        eng.check()
        assert int(eng.peer_epoch.item()) == len(forced)
    assert runs[0] == runs[1]


def test_engine_push_over_torch_symmetric_memory():
    """The accumulators in torch symmetric memory (one-rank NCCL group in a worker process): the buffer and the peer
    offsets are obtained the way a multi-GPU run obtains them."""
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_tp_graph_worker.py")
    r = subprocess.run([sys.executable, worker, "push", str(port)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "TP_PUSH_SYMM_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


def test_peer_bcast_and_argmax_between_two_streams(af):
    """`af_peer_bcast` (rank 0's decision record into every rank's slot) and `af_peer_argmax` (every rank's (value, index)
    pair to every rank; largest value, lowest index on ties) with two streams playing the ranks over two regions of
    one allocation, three rounds (the counters are monotonic; the epochs live on the device)."""
    from paper_2603_11873_b200.adapters import peer_argmax, peer_bcast

    tp = 2
    region = 64                                              # int64 words per rank: counters | 16-word slot | pair slots
    shared = torch.zeros(tp * region, dtype=torch.int64, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(tp)]
    epochs = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(tp)]
    regs = [shared[r * region: (r + 1) * region] for r in range(tp)]
    offs = [[(q - r) * region * 8 for q in range(tp)] for r in range(tp)]
    src = torch.zeros(3, 16, dtype=torch.int64, device="cuda")
    for rnd in range(3):
        src[rnd] = torch.arange(16, device="cuda") * 7 + rnd * 1000 + 1
    dst = [torch.zeros(3, 16, dtype=torch.int64, device="cuda") for _ in range(tp)]
    # round -> (values, indices) per rank; round 1 is a tie in value: the lower index wins
    vals = [[1.5, 2.5], [3.0, 3.0], [-1.0, -2.0]]
    idxs = [[7, 300], [400, 9], [5, 600]]
    want = [300, 9, 5]
    val_t = [[torch.tensor([vals[rnd][r]], dtype=torch.float32, device="cuda") for r in range(tp)] for rnd in range(3)]
    idx_t = [[torch.tensor([idxs[rnd][r]], dtype=torch.int32, device="cuda") for r in range(tp)] for rnd in range(3)]
    out = [torch.zeros(3, dtype=torch.int32, device="cuda") for _ in range(tp)]
    torch.cuda.synchronize()
    for rnd in range(3):
        for r in range(tp):                                  # (calls that wait for each other are enqueued back to back)
            with torch.cuda.stream(streams[r]):
                c32 = regs[r][:1].view(torch.int32)
                peer_bcast(src[rnd] if r == 0 else None, regs[r][2:18], dst[r][rnd], r == 0, c32[0:1], epochs[r][0:1], offs[r])
        for r in range(tp):
            with torch.cuda.stream(streams[r]):
                c32 = regs[r][:1].view(torch.int32)
                peer_argmax(val_t[rnd][r], idx_t[rnd][r], regs[r][18:26], r, c32[1:2], epochs[r][1:2], offs[r], out[r][rnd: rnd + 1])
    torch.cuda.synchronize()
    for r in range(tp):
        assert torch.equal(dst[r], src), r
        assert out[r].tolist() == want, (r, out[r].tolist())
        assert epochs[r].tolist() == [3, 3]
        assert regs[r][:1].view(torch.int32).tolist() == [3, 3 * tp]     # one bump per broadcast (the root's), tp per gather


def test_single_phase_group_with_peers_needs_its_counter(af):
    """A one-projection group whose only phase is pushed to the peers reports on phase_done[0]; without counters the
    launch is refused before anything runs."""
    from paper_2603_11873_b200.adapters import SegmentGroup

    shapes, w, down, up = _full_model(seed=14)
    tg, tab = _table(w, down, up)
    grp = SegmentGroup(tab, [0])
    grp.set_peers([0], reduce_phases=[0])
    acc = torch.zeros(D, dtype=torch.int64, device="cuda")
    x = torch.ones(D, device="cuda")
    cur = _decision((1, 2), (0.5, 0.5))
    with pytest.raises(Exception):
        grp.switch_gemv(None, cur, acc, xin=x, max_k=2)                     # no counters at all
    done = torch.zeros(1, dtype=torch.int32, device="cuda")
    grp.switch_gemv_chain(None, cur, [dict(acc_out=acc, xin=x)], done, max_k=2)
    tab.status()
    assert done.item() == grp.grid and float(acc.abs().max()) > 0


def test_a_missing_peer_times_out_and_later_waits_fail_fast(af):
    """A wait for a peer that never arrives raises AF_ECUDA in the caller's status word after ~2 s instead of hanging; with
    the word already set, later waits give up after ~2 ms each -- a dead rank fails a step in seconds, not minutes."""
    import time

    from paper_2603_11873_b200 import _capi
    from paper_2603_11873_b200.adapters import peer_barrier, peer_wait

    counter = torch.zeros(2, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    t0 = time.time()
    peer_wait(counter[0:1], 1, err)                              # nobody bumps it
    torch.cuda.synchronize()
    first = time.time() - t0
    # (2^32 SM cycles: 2.2 s at 1965 MHz, longer if the clocks have not ramped up for a one-thread kernel)
    assert err.item() == _capi.AF_ECUDA and 1.0 < first < 90.0, (err.item(), first)
    t0 = time.time()
    for _ in range(20):
        peer_wait(counter[0:1], 1, err)
    epoch = torch.zeros(1, dtype=torch.int32, device="cuda")
    peer_barrier(counter[1:2], epoch, [0, 8], err)               # a "second rank" (the next word) that never joins
    torch.cuda.synchronize()
    later = time.time() - t0
    assert later < max(1.0, first / 2), (later, first)            # 21 waits of ~2 ms (2^22 cycles) each, not 21 time-outs
    assert counter[1].item() == 1 and epoch.item() == 1          # this rank did its part of the barrier
