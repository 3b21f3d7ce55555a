"""Pin the CPU oracle (oracle/) against the reference.

Two anchors:
  (a) golden values that live in the reference's own tests, restated literally here
      with the file:line they come from (/root/reference/pkg/tests/...);
  (b) fixtures produced by running the unmodified reference (tests/golden/make_golden.py).
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import oracle as orc


# ------------------------------------------------------------------ (a) ------


class TestReferenceTestVectors:
    def test_router_worked_example(self):
        # tests/test_routing.py:17-23
        ids, w, logits = orc.route([[1.0, 0.0], [0.0, 1.0], [0.0, 0.0]], [2.0, 1.0], 2)
        assert ids == (0, 1)
        assert abs(w[0] - 0.73106) <= 1e-5 and abs(w[1] - 0.26894) <= 1e-5
        assert list(logits) == [2.0, 1.0, 0.0]

    def test_router_zero_vector_ties(self):
        # tests/test_routing.py:25-29
        ids, w, _ = orc.route(np.ones((4, 3)), [0.0, 0.0, 0.0], 2)
        assert ids == (0, 1) and w == (0.5, 0.5)

    def test_router_tie_order_ascending_index(self):
        # tests/test_routing.py:61-64
        ids, _, _ = orc.route([[1.0], [1.0], [1.0]], [1.0], 3)
        assert ids == (0, 1, 2)

    def test_router_signed_zero_ties(self):
        # +0.0 and -0.0 compare equal, index order decides
        ids, _, _ = orc.route([[1.0], [-1.0], [1.0]], [0.0], 2)
        assert ids == (0, 1)

    @pytest.mark.parametrize("k", [0, -1, 4])
    def test_router_rejects_k(self, k):
        # tests/test_routing.py:102-105
        with pytest.raises(ValueError):
            orc.route(np.eye(3), [1.0, 2.0, 3.0], k)

    def test_router_invariants(self):
        # tests/test_routing.py:42-59 (f32 restatement: sum to 1 within f32 round-off)
        rng = np.random.Generator(np.random.PCG64(22))
        wg = rng.uniform(-1, 1, (8, 16)).astype(np.float32)
        for _ in range(300):
            k = int(rng.integers(1, 9))
            x = rng.normal(size=16).astype(np.float32)
            ids, w, logits = orc.route(wg, x, k)
            assert len(set(ids)) == k and all(v > 0 for v in w)
            assert abs(sum(w) - 1.0) <= 1e-6
            picked = [logits[i] for i in ids]
            assert all(a >= b for a, b in zip(picked, picked[1:]))
            rest = [l for i, l in enumerate(logits) if i not in ids]
            if rest:
                assert min(picked) >= max(rest)

    def test_rank_one_update_example(self):
        # tests/test_linalg.py:120-126
        c = np.eye(2, dtype=np.float32)
        orc.gemm_accumulate(c, [[1.0], [0.0]], [[1.0, 0.0]], +1)
        assert np.array_equal(c, [[2.0, 0.0], [0.0, 1.0]])

    def test_sgmm_two_segment_example(self):
        # tests/test_linalg.py:161-174
        t1 = np.eye(2, dtype=np.float32)
        t2 = np.eye(2, dtype=np.float32)
        orc.sgmm_segment(t1, [[1.0], [0.0]], [[1.0, 0.0]], +1)
        orc.sgmm_segment(t2, [[0.0], [1.0]], [[0.0, 1.0]], +1)
        assert np.array_equal(t1, [[2.0, 0.0], [0.0, 1.0]])
        assert np.array_equal(t2, [[1.0, 0.0], [0.0, 2.0]])

    def test_sgmm_zero_rank_is_noop(self):
        # tests/test_linalg.py:226-231
        t = np.eye(3, dtype=np.float32)
        orc.sgmm_segment(t, np.zeros((3, 0)), np.zeros((0, 3)), +1)
        assert np.array_equal(t, np.eye(3))

    def test_sgmm_rejects_bad_sign(self):
        with pytest.raises(ValueError):
            orc.sgmm_segment(np.zeros((2, 2), np.float32), np.zeros((2, 1)), np.zeros((1, 2)), 2)

    def test_sgmm_round_trip(self):
        # tests/test_linalg.py:209-217 (f32 band)
        rng = np.random.Generator(np.random.PCG64(12))
        t = rng.uniform(-1, 1, (32, 32)).astype(np.float32)
        before = t.copy()
        up = rng.uniform(-1, 1, (32, 8)).astype(np.float32)
        down = rng.uniform(-1, 1, (8, 32)).astype(np.float32)
        orc.sgmm_segment(t, up, down, +1)
        orc.sgmm_segment(t, up, down, -1)
        assert np.max(np.abs(t - before)) <= 2e-6

    def test_golden_weight_digest(self, golden):
        # tests/test_model.py:30-33, 103-109: seed-42 single-precision digest
        want = "1e7b53f3962d8d8838a86517adfdaf96696437371056c6a9ecd5eb2b8795d1ae"
        assert bytes(golden("generate")["digest_single_seed42"]).decode() == want
        m = orc.build_toy_model(orc.ToyConfig(layers=4, hidden=8, vocab=16, experts=4, rank=2, top_k=2, seed=42), bf16=False)
        h = hashlib.sha256()
        h.update(m.embed.tobytes()); h.update(m.router.tobytes()); h.update(m.unembed.tobytes())
        for li in range(4):
            h.update(m.pristine[li].tobytes())
            for e in range(4):
                h.update(m.down_bank[li][e].tobytes()); h.update(m.up_bank[li][e].tobytes())
        assert h.hexdigest() == want


# ------------------------------------------------------------------ (b) ------


class TestAgainstReferenceRuns:
    def test_router_cases(self, golden):
        g = golden("router")
        for i in range(int(g["n_cases"])):
            ids, w, logits = orc.route(g[f"c{i}_wg"], g[f"c{i}_x"], int(g[f"c{i}_k"]))
            assert ids == tuple(int(v) for v in g[f"c{i}_ids"]), f"case {i} margin {float(g[f'c{i}_margin'])}"
            assert np.allclose(w, g[f"c{i}_weights"], rtol=2e-6, atol=1e-7)
            # reference logits come from OpenBLAS sgemv; ours are the correctly rounded dot
            assert np.allclose(logits, g[f"c{i}_logits"], rtol=0, atol=2e-6 * max(1.0, float(np.abs(logits).max())))

    def test_sgmm_bit_exact(self, golden):
        g = golden("sgmm")
        for i in range(int(g["n_cases"])):
            for sign, tag in ((+1, "p"), (-1, "m")):
                t = g[f"s{i}_target"].copy()
                orc.sgmm_segment(t, g[f"s{i}_up"], g[f"s{i}_down"], sign)
                assert np.array_equal(t, g[f"s{i}_after_{tag}"]), f"case {i} sign {sign}"

    def test_gemm_accumulate_close(self, golden):
        # BLAS summation order differs: few f32 ulp
        g = golden("sgmm")
        for i in range(int(g["n_cases"])):
            t = g[f"s{i}_target"].copy()
            orc.gemm_accumulate(t, g[f"s{i}_up"], g[f"s{i}_down"], +1)
            assert np.allclose(t, g[f"s{i}_gai_p"], rtol=0, atol=3e-7)

    def test_switch_sequence_bit_exact(self, golden):
        g = golden("switch")
        n_layers = int(g["n_layers"])
        w = [g[f"w{li}"].copy() for li in range(n_layers)]
        prev = None
        for t in range(int(g["n_tokens"])):
            cur = (tuple(int(v) for v in g[f"t{t}_ids"]), tuple(float(v) for v in g[f"t{t}_weights"]))
            for li in range(n_layers):
                down_cat, up_cat = orc.switch_factors(g[f"down{li}"], g[f"up{li}"], prev, cur)
                if t == 1 and li == 0:
                    assert np.array_equal(down_cat, g["sw1_down0"]) and np.array_equal(up_cat, g["sw1_up0"])
                orc.sgmm_segment(w[li], up_cat, down_cat, +1)
                assert np.array_equal(w[li], g[f"t{t}_w{li}"]), f"token {t} layer {li}"
            prev = cur
        for li in range(n_layers):
            down_cat, up_cat = orc.switch_factors(g[f"down{li}"], g[f"up{li}"], None, prev)
            orc.sgmm_segment(w[li], up_cat, down_cat, -1)
            assert np.array_equal(w[li], g[f"final_w{li}"])

    @pytest.mark.parametrize("name", ["c1", "c1v1024", "small"])
    def test_generate_f32_matches_reference(self, golden, name):
        g = golden("generate")
        L, d, V, N, r, k, seed = (int(v) for v in g[f"{name}_config"])
        cfg = orc.ToyConfig(layers=L, hidden=d, vocab=V, experts=N, rank=r, top_k=k, seed=seed)
        # greedy generate()
        model = orc.build_toy_model(cfg, bf16=True)
        sink = []
        n_new = len(g[f"{name}_greedy_tokens"])
        toks, _, _ = orc.toy_generate(model, [7, 42, 3], n_new, storage="f32", hidden_sink=sink)
        assert toks == [int(v) for v in g[f"{name}_greedy_tokens"]]
        hid = np.stack([s[-1] for s in sink])
        assert np.max(np.abs(hid - g[f"{name}_greedy_hidden_last"])) <= 1e-5
        dev = max(float(np.max(np.abs(a - b))) for a, b in zip(model.backbone, model.pristine))
        # same residue as the reference's own run (a repeated token drifts linearly in f32)
        assert abs(dev - float(g[f"{name}_restore_dev"])) <= 2e-7
        # teacher-forced stream: ids bit-exact, weights/logits within f32 round-off
        model = orc.build_toy_model(cfg, bf16=True)
        forced = g[f"{name}_forced_tokens"]
        toks, logits, decs = orc.toy_generate(model, [int(forced[0])], len(forced), storage="f32", forced=forced)
        assert toks == [int(v) for v in g[f"{name}_forced_next"]]
        for t, (ids, w) in enumerate(decs):
            assert ids == tuple(int(v) for v in g[f"{name}_forced_ids"][t])
            assert np.allclose(w, g[f"{name}_forced_weights"][t], rtol=2e-6)
        ref_logits = g[f"{name}_forced_logits"]
        assert np.max(np.abs(np.stack(logits) - ref_logits)) <= 1e-5 * max(1.0, float(np.abs(ref_logits).max()))

    def test_bf16_storage_stays_within_one_ulp_of_f32_path(self, golden):
        """The bf16 per-step oracle equals the f32 switch on the upcast weights, rounded:
        one step from pristine must equal round_bf16(f32 result) exactly."""
        g = golden("generate")
        L, d, V, N, r, k, seed = (int(v) for v in g["small_config"])
        cfg = orc.ToyConfig(layers=L, hidden=d, vocab=V, experts=N, rank=r, top_k=k, seed=seed)
        a = orc.build_toy_model(cfg)
        b = orc.build_toy_model(cfg)
        orc.toy_decode_step(a, orc.ToyState(), 5, storage="f32")
        orc.toy_decode_step(b, orc.ToyState(), 5, storage="bf16")
        for li in range(L):
            assert np.array_equal(orc.to_bf16_bits(a.backbone[li]), b.backbone_bits[li])


class TestBf16Helpers:
    def test_round_trip_and_rne(self):
        import torch

        rng = np.random.Generator(np.random.PCG64(3))
        x = (rng.normal(size=4096) * np.exp(rng.uniform(-20, 20, 4096))).astype(np.float32)
        want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        assert np.array_equal(orc.to_bf16_bits(x), want)
        assert np.array_equal(orc.round_bf16(orc.round_bf16(x)), orc.round_bf16(x))

    def test_ulp_distance(self):
        a = orc.to_bf16_bits(np.array([1.0, -1.0, 0.0, 2.0], np.float32))
        b = a.copy()
        b[0] += 1
        b[3] -= 2
        assert orc.max_ulp_diff_bf16(a, b) == (2, 2)


def test_oracle_thread_override_under_torchrun_env():
    """torchrun exports OMP_NUM_THREADS=1; the timed baseline (bench.py cpu_sample) must still get
    the host's cores by asking for them explicitly."""
    import subprocess
    import sys

    code = ("from oracle import oracle as o\n"
            "assert o.num_threads() == 1, o.num_threads()\n"
            "o.set_num_threads(4)\n"
            "assert o.num_threads() == 4, o.num_threads()\n")
    env = dict(os.environ, OMP_NUM_THREADS="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_ulp_report_c_pass_equals_numpy():
    """oracle.strict_ulp_report (one OpenMP pass in oracle.c, what the true-shape GPU tests call on 45M-element
    matrices) against its plain numpy statement."""
    rng = np.random.default_rng(0)
    want = orc.to_bf16_bits(rng.normal(size=(300, 257)).astype(np.float32) * 0.01)
    got = want.copy()
    idx = rng.integers(0, want.size, 2000)
    got.reshape(-1)[idx] += rng.integers(-3, 4, 2000).astype(np.uint16)
    got.reshape(-1)[7] = want.reshape(-1)[7] ^ 0x8000 if want.reshape(-1)[7] & 0x7FFF == 0 else got.reshape(-1)[7]
    r1 = orc.to_bf16_bits(rng.normal(size=want.shape).astype(np.float32) * 0.05)
    r2 = orc.to_bf16_bits(rng.normal(size=want.shape).astype(np.float32) * 0.001)
    a, b = orc.strict_ulp_report(got, want, r1, r2), orc.strict_ulp_report_numpy(got, want, r1, r2)
    assert a["n"] == b["n"] and a["n_diff"] == b["n_diff"] and a["n_violations"] == b["n_violations"]
    for k in ("max_strict", "max_relaxed", "worst_ratio"):
        assert abs(a[k] - b[k]) <= 1e-12 * max(1.0, abs(b[k])), k
    same = orc.strict_ulp_report(want, want, r1)
    assert same["n_diff"] == 0 and same["max_strict"] == 0.0 and same["n_violations"] == 0
