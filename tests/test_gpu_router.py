"""Router parity on the GPU: `af_pregate` (through the Python mirror of routing.py) against
the CPU oracle and the fixtures generated from the unmodified reference.  Expert ids must be
bit-exact (BASELINE.json north_star)."""

import numpy as np
import pytest
import torch

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def af():
    import paper_2603_11873_b200 as af

    return af


def _route_gpu(af, wg, x, k, wprec="bf16", xprec="single"):
    router = af.RouterParams(weight=af.Matrix(np.asarray(wg, np.float32), wprec))
    xm = af.Matrix(np.asarray(x, np.float32).reshape(-1, 1), xprec)
    rec = af.DispatchRecorder()
    dec = af.route(router, xm, k, rec)
    return dec, rec


def test_golden_router_cases(af, golden):
    g = golden("router")
    n = int(g["n_cases"])
    risky = 0
    for i in range(n):
        wg, x, k = g[f"c{i}_wg"], g[f"c{i}_x"], int(g[f"c{i}_k"])
        dec, _ = _route_gpu(af, wg, x, k)
        o_ids, o_w, _ = orc.route(wg, x, k)
        assert dec.expert_ids == o_ids, f"case {i}: ids differ from the oracle"
        np.testing.assert_allclose(dec.weights, o_w, rtol=2e-6, atol=1e-7)
        if float(g[f"c{i}_margin"]) > 1e-6:  # OpenBLAS summation-order noise is ~1e-8
            assert dec.expert_ids == tuple(int(v) for v in g[f"c{i}_ids"]), f"case {i}: ids differ from the reference"
            np.testing.assert_allclose(dec.weights, g[f"c{i}_weights"], rtol=1e-5, atol=1e-7)
        else:
            risky += 1
    assert risky < n // 4


def test_reference_worked_examples(af):
    # /root/reference/pkg/tests/test_routing.py:17-29, :61-64
    dec, rec = _route_gpu(af, [[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]], [2.0, 1.0], 2)
    assert dec.expert_ids == (0, 1)
    assert abs(dec.weights[0] - 0.73106) <= 1e-5 and abs(dec.weights[1] - 0.26894) <= 1e-5
    assert [e.kind for e in rec.events] == ["gemm", "elementwise"] and all(e.label == "router" for e in rec.events)
    dec, _ = _route_gpu(af, np.ones((4, 3)), [0.0, 0.0, 0.0], 2)
    assert dec.expert_ids == (0, 1) and dec.weights == (0.5, 0.5)
    dec, _ = _route_gpu(af, [[1.0], [1.0], [1.0]], [1.0], 3)
    assert dec.expert_ids == (0, 1, 2)
    dec, _ = _route_gpu(af, [[1.0], [-1.0], [1.0]], [0.0], 2)  # +0.0 / -0.0 tie -> index order
    assert dec.expert_ids == (0, 1)


@pytest.mark.parametrize("wprec,xprec", [("bf16", "single"), ("single", "single"), ("bf16", "bf16"), ("single", "bf16")])
def test_random_vectors_bit_exact_ids(af, wprec, xprec):
    rng = np.random.Generator(np.random.PCG64(77))
    for n, d, k in [(8, 256, 2), (16, 4096, 2), (8, 8192, 4), (5, 37, 5), (64, 130, 8), (256, 64, 3)]:
        wg = orc.round_bf16(rng.uniform(-1, 1, (n, d)).astype(np.float32) / np.sqrt(d))
        for _ in range(8):
            x = orc.round_bf16(rng.normal(size=d).astype(np.float32))
            dec, _ = _route_gpu(af, wg, x, k, wprec, xprec)
            ids, w, _ = orc.route(wg, x, k)
            assert dec.expert_ids == ids
            np.testing.assert_allclose(dec.weights, w, rtol=2e-6, atol=1e-7)
            assert abs(sum(dec.weights) - 1.0) < 1e-6 and all(v > 0 for v in dec.weights)


def test_logits_match_oracle_bitwise(af):
    rng = np.random.Generator(np.random.PCG64(5))
    wg = orc.round_bf16(rng.uniform(-1, 1, (16, 4096)).astype(np.float32) / 64)
    x = orc.round_bf16(rng.normal(size=4096).astype(np.float32))
    router = af.RouterParams(weight=af.Matrix(wg, "bf16"))
    got = af.router_logits(router, af.Matrix(x.reshape(-1, 1), "single"))
    _, _, want = orc.route(wg, x, 1)
    assert np.array_equal(got, want)  # correctly rounded f32 dot products on both sides


def test_errors(af):
    router = af.RouterParams(weight=af.Matrix(np.eye(3, dtype=np.float32), "bf16"))
    x = af.Matrix(np.ones((3, 1), np.float32), "single")
    for k in (0, -1, 4):  # tests/test_routing.py:102-105
        with pytest.raises(ValueError):
            af.route(router, x, k, af.DispatchRecorder())
    with pytest.raises(af.DimensionError):  # tests/test_routing.py:106-109
        af.route(router, af.Matrix(np.ones((4, 1), np.float32), "single"), 1, af.DispatchRecorder())
    with pytest.raises(af.DimensionError):
        af.route(router, af.Matrix(np.ones((1, 3), np.float32), "single"), 1, af.DispatchRecorder())


def test_device_decision_round_trip(af):
    gd = af.GateDecision((3, 1), (0.75, 0.25))
    dd = af.DeviceDecision.from_host(gd)
    assert dd.to_host() == gd
    assert torch.cuda.is_available()


def test_nan_logits_sort_last_like_numpy(af):
    """routing.py:64-65 is `np.argsort(-logits, kind="stable")`: numpy sorts NaN after every number (and NaN against NaN
    by index).  A router row that produces NaN must therefore never be selected while k numbers exist."""
    import torch

    n, d, k = 8, 64, 3
    rng = np.random.Generator(np.random.PCG64(77))
    w = rng.uniform(-1, 1, (n, d)).astype(np.float32)
    x = rng.uniform(-1, 1, d).astype(np.float32)
    w[0, 5] = np.nan            # the very first expert: "first seen in a lane" must not stick as the lane's best
    w[6, 1] = np.nan
    router = af.RouterParams(weight=af.Matrix(torch.from_numpy(w).cuda(), "single"))
    dec = af.route(router, af.Matrix(torch.from_numpy(x.reshape(-1, 1)).cuda(), "single"), k, af.DispatchRecorder())
    logits = (w.astype(np.float64) @ x.astype(np.float64)).astype(np.float32)
    want = tuple(int(i) for i in np.argsort(-logits, kind="stable")[:k])
    assert 0 not in dec.expert_ids and 6 not in dec.expert_ids
    assert dec.expert_ids == want
    # with fewer than k numbers the NaN rows fill the tail, lowest index first
    w2 = np.full((4, d), np.nan, np.float32)
    w2[2] = rng.uniform(-1, 1, d)
    router2 = af.RouterParams(weight=af.Matrix(torch.from_numpy(w2).cuda(), "single"))
    dec2 = af.route(router2, af.Matrix(torch.from_numpy(x.reshape(-1, 1)).cuda(), "single"), 3, af.DispatchRecorder())
    assert dec2.expert_ids == (2, 0, 1)
