"""Generate the committed golden fixtures by running the UNMODIFIED reference.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `lorafuse` from /root/reference/pkg/src, feeds it seeded inputs in
precision "single" (weights optionally pre-rounded to the bf16 grid -- the 'bf16 shim'
of SURVEY.md section 7 step 1, so the reference does f32 arithmetic on bf16-representable
inputs) and stores inputs + outputs as small .npz files next to this script.  The tests
replay the same inputs through oracle/ (CPU) and through the CUDA path (GPU).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import lorafuse as lf  # noqa: E402
from lorafuse import adapters as lfa  # noqa: E402
from lorafuse import model as lfm  # noqa: E402


def bf16_round(a: np.ndarray) -> np.ndarray:
    """RNE f32 -> bf16 grid, carried as f32 (independent of oracle/ on purpose)."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    lsb = (u >> 16) & 1
    r = (u + 0x7FFF + lsb) & 0xFFFF0000
    return r.astype(np.uint32).view(np.float32)


def single(a) -> lf.Matrix:
    return lf.Matrix(np.asarray(a, dtype=np.float32), "single")


# ---------------------------------------------------------------- router ----


def golden_router():
    rng = np.random.Generator(np.random.PCG64(1001))
    cases = []
    for n, d, k in [(8, 256, 2), (8, 64, 2), (16, 512, 2), (8, 1024, 4), (5, 6, 5), (3, 7, 1), (16, 4096, 2)]:
        for _ in range(12 if n * d <= 8192 else 3):
            wg = bf16_round(rng.uniform(-1, 1, (n, d)).astype(np.float32) / np.sqrt(d))
            x = bf16_round(rng.normal(size=d).astype(np.float32))
            dec = lf.route(lf.RouterParams(weight=single(wg)), single(x.reshape(-1, 1)), k, lf.DispatchRecorder())
            logits = (single(wg).data @ x.reshape(-1, 1))[:, 0]
            srt = np.sort(logits)[::-1]
            margin = float(np.min(srt[:k] - srt[1 : k + 1])) if k < n else float(np.min(-np.diff(srt)))
            cases.append(dict(wg=wg, x=x, k=k, ids=np.array(dec.expert_ids, np.int32),
                              weights=np.array(dec.weights, np.float64), logits=logits, margin=margin))
    out = {}
    for i, c in enumerate(cases):
        for key, v in c.items():
            out[f"c{i}_{key}"] = np.asarray(v)
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "router.npz"), **out)
    print("router.npz:", len(cases), "cases; min margin", min(c["margin"] for c in cases))


# ------------------------------------------------------------------ sgmm ----


def golden_sgmm():
    rng = np.random.Generator(np.random.PCG64(1002))
    out = {}
    shapes = [(33, 29, 9), (64, 64, 32), (48, 200, 16), (130, 72, 5), (8, 8, 1), (16, 40, 0), (256, 256, 32)]
    for i, (d_out, d_in, s) in enumerate(shapes):
        tgt = bf16_round(rng.uniform(-0.125, 0.125, (d_out, d_in)).astype(np.float32))
        up = bf16_round(rng.uniform(-0.5, 0.5, (d_out, s)).astype(np.float32))
        down = rng.uniform(-0.1, 0.1, (s, d_in)).astype(np.float32)  # NOT bf16: gate-folded factors are f32
        for sign in (+1, -1):
            t = single(tgt.copy())
            table = lf.SegmentTable([lf.Segment(single(down), single(up), t)])
            lf.sgmm(table, sign, lf.DispatchRecorder())
            out[f"s{i}_after_{'p' if sign > 0 else 'm'}"] = t.data.copy()
        t = single(tgt.copy())
        lf.gemm_accumulate_inplace(t, single(up), single(down), +1, lf.DispatchRecorder())
        out[f"s{i}_gai_p"] = t.data.copy()
        out[f"s{i}_target"], out[f"s{i}_up"], out[f"s{i}_down"] = tgt, up, down
    out["n_cases"] = np.array(len(shapes))
    np.savez_compressed(os.path.join(HERE, "sgmm.npz"), **out)
    print("sgmm.npz:", len(shapes), "cases")


# ---------------------------------------------------------------- switch ----


def golden_switch():
    """concat_gated + build_switch + merge_all on a small bank, two consecutive tokens."""
    rng = np.random.Generator(np.random.PCG64(1003))
    n_layers, n_exp, r, d_out, d_in = 3, 6, 4, 40, 56
    out = {}
    backbone, layers = [], []
    for li in range(n_layers):
        w = bf16_round(rng.uniform(-0.125, 0.125, (d_out, d_in)).astype(np.float32))
        backbone.append(single(w.copy()))
        out[f"w{li}"] = w
        experts = []
        downs, ups = [], []
        for _ in range(n_exp):
            dn = bf16_round(rng.uniform(-0.2, 0.2, (r, d_in)).astype(np.float32))
            up = bf16_round(rng.uniform(-0.5, 0.5, (d_out, r)).astype(np.float32))
            experts.append(lf.LoraExpert(down=single(dn), up=single(up)))
            downs.append(dn)
            ups.append(up)
        layers.append(tuple(experts))
        out[f"down{li}"] = np.stack(downs)
        out[f"up{li}"] = np.stack(ups)
    gates = [
        lf.GateDecision((4, 1), (float(np.float32(0.7)), float(np.float32(0.3)))),
        lf.GateDecision((1, 5), (float(np.float32(0.55)), float(np.float32(0.45)))),
        lf.GateDecision((1, 5), (float(np.float32(0.55)), float(np.float32(0.45)))),
        lf.GateDecision((0, 2), (float(np.float32(0.9)), float(np.float32(0.1)))),
    ]
    prev = None
    rec = lf.DispatchRecorder()
    for t, gate in enumerate(gates):
        cur = [lfa.concat_gated(layer, gate) for layer in layers]
        sw = cur if prev is None else [lfa.build_switch(p, c) for p, c in zip(prev, cur)]
        if t == 1:
            out["sw1_down0"] = sw[0].down_cat.data.copy()
            out["sw1_up0"] = sw[0].up_cat.data.copy()
        lf.merge_all(backbone, sw, +1, rec)
        for li in range(n_layers):
            out[f"t{t}_w{li}"] = backbone[li].data.copy()
        out[f"t{t}_ids"] = np.array(gate.expert_ids, np.int32)
        out[f"t{t}_weights"] = np.array(gate.weights, np.float32)
        prev = cur
    lf.merge_all(backbone, prev, -1, rec)
    for li in range(n_layers):
        out[f"final_w{li}"] = backbone[li].data.copy()
    out["n_tokens"] = np.array(len(gates))
    out["n_layers"] = np.array(n_layers)
    np.savez_compressed(os.path.join(HERE, "switch.npz"), **out)
    print("switch.npz: sgmm events", rec.counts()["sgmm"])


# -------------------------------------------------------------- generate ----


def shim_model_to_bf16(model):
    """Round every weight of a reference model to the bf16 grid, in place (f32 carrier)."""
    for m in [model.embed, model.router.weight, model.unembed, *model.backbone, *model.pristine_backbone]:
        m.data[...] = bf16_round(m.data)
    for layer in model.bank.layers:
        for e in layer:
            e.down.data[...] = bf16_round(e.down.data)
            e.up.data[...] = bf16_round(e.up.data)


def golden_generate():
    out = {}
    configs = {
        "c1": dict(layers=4, hidden=256, vocab=256, experts=8, rank=8, top_k=2, seed=0),
        "c1v1024": dict(layers=4, hidden=256, vocab=1024, experts=8, rank=8, top_k=2, seed=2),
        "small": dict(layers=3, hidden=64, vocab=64, experts=4, rank=4, top_k=2, seed=5),
    }
    for name, kw in configs.items():
        n_new = 64 if name != "small" else 16
        cfg = lf.ModelConfig(precision="single", strategy=lf.Strategy.PRE_GATED_FUSED, **kw)
        # (1) greedy generate(), exactly what the reference API does
        model = lf.build_model(cfg)
        shim_model_to_bf16(model)
        sink = []
        toks, trace = lf.generate(model, [7, 42, 3], n_new, lf.DispatchRecorder(), hidden_sink=sink)
        out[f"{name}_greedy_tokens"] = np.array(toks, np.int32)
        out[f"{name}_greedy_hidden_last"] = np.stack([np.asarray(s[-1], np.float32) for s in sink])
        out[f"{name}_restore_dev"] = np.array(lf.max_backbone_deviation(model))
        out[f"{name}_sgmm_events"] = np.array(sum(1 for ev in trace if ev.kind == "sgmm"))
        # (2) teacher-forced stream through decode_step: every step switches
        model = lf.build_model(cfg)
        shim_model_to_bf16(model)
        forced = np.random.Generator(np.random.PCG64(kw["seed"] + 1)).integers(0, kw["vocab"], n_new)
        state = lfm.DecodeState()
        rec = lf.DispatchRecorder()
        nxt, ids, wts, hid, logit_rows, margins = [], [], [], [], [], []
        for tkn in forced:
            x = lfm._embed_token(model, int(tkn), lf.DispatchRecorder())
            lg = (model.router.weight.data @ x.data)[:, 0]
            srt = np.sort(lg)[::-1]
            margins.append(float(np.min(srt[: cfg.top_k] - srt[1 : cfg.top_k + 1])))
            cap = []
            t_next, _ = lf.decode_step(model, state, int(tkn), rec, capture=cap)
            nxt.append(t_next)
            gate = state.prev_concats[0].provenance
            ids.append([p[0] for p in gate])
            wts.append([p[1] for p in gate])
            hid.append(np.asarray(cap[-1], np.float32))
            logit_rows.append((hid[-1].reshape(1, -1) @ model.unembed.data)[0])
        out[f"{name}_forced_tokens"] = np.asarray(forced, np.int32)
        out[f"{name}_forced_next"] = np.array(nxt, np.int32)
        out[f"{name}_forced_ids"] = np.array(ids, np.int32)
        out[f"{name}_forced_weights"] = np.array(wts, np.float32)
        out[f"{name}_forced_hidden_last"] = np.stack(hid)
        out[f"{name}_forced_logits"] = np.stack(logit_rows).astype(np.float32)
        out[f"{name}_forced_margin"] = np.array(margins)
        out[f"{name}_forced_w0_after"] = model.backbone[0].data.copy()
        lf.finalize_generation(model, state, rec)
        out[f"{name}_forced_restore_dev"] = np.array(lf.max_backbone_deviation(model))
        out[f"{name}_config"] = np.array([kw[k] for k in ("layers", "hidden", "vocab", "experts", "rank", "top_k", "seed")])
        print(name, "greedy distinct", len(set(toks)), "forced min margin", min(margins),
              "restore dev", float(out[f"{name}_forced_restore_dev"]))
    # weight identity: digests for the reference's own golden config (tests/test_model.py:30-33)
    cfg = lf.ModelConfig(layers=4, hidden=8, vocab=16, experts=4, rank=2, top_k=2, precision="single", seed=42)
    out["digest_single_seed42"] = np.frombuffer(lf.weights_digest(lf.build_model(cfg)).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "generate.npz"), **out)


def golden_io():
    """Containers written by the reference's OWN save_bank / save_checkpoint (adapters.py:265-306,
    model.py:481-541) for a small bf16-shimmed model, plus what the reference decodes from it: the
    loaders of the B200 package must read these files and reproduce the tokens."""
    kw = dict(layers=2, hidden=32, vocab=48, experts=4, rank=8, top_k=2, seed=7)
    model = lf.build_model(lf.ModelConfig(precision="single", strategy=lf.Strategy.PRE_GATED_FUSED, **kw))
    shim_model_to_bf16(model)
    lfa.save_bank(model.bank, os.path.join(HERE, "ref_bank.npz"))
    lfm.save_checkpoint(model, os.path.join(HERE, "ref_checkpoint.npz"))
    rec = lf.DispatchRecorder()
    toks, _ = lf.generate(model, [3, 11, 40], 10, rec)
    np.savez(os.path.join(HERE, "ref_io_expected.npz"), tokens=np.array(toks, np.int32), digest=np.frombuffer(
        lf.weights_digest(model).encode(), dtype=np.uint8), config=np.array([kw[k] for k in ("layers", "hidden", "vocab", "experts", "rank", "top_k", "seed")]))
    print("io fixtures: tokens", toks)


def golden_harness():
    """Reports written by the reference's OWN harness (cli.py) on a small single-precision config:
    the bench report + CSV, the profile document and the seeded workload; plus known answers of
    perf.estimate / breakdown / calibrate on a hand-made trace.  The B200 harness must reproduce
    every field that is a function of the dispatch trace (counts, flops, estimated ms)."""
    import json

    from lorafuse import cli as lfc
    from lorafuse import perf as lfp
    from lorafuse.linalg import DispatchEvent

    os.environ["SOURCE_DATE_EPOCH"] = "0"
    cfg_text = ("layers: 3\nhidden: 64\nvocab: 128\nexperts: 4\nrank: 4\ntop_k: 2\nprecision: single\nseed: 5\n"
                "launch_seconds: 1.0e-5\nflops_throughput: 1.0e+10\nbytes_bandwidth: 2.0e+9\n"
                "n_new: 6\nsynthetic_prompts: 3\nsynthetic_len_min: 2\nsynthetic_len_max: 5\n")
    cfg_path = os.path.join(HERE, "ref_harness_config.yaml")
    with open(cfg_path, "w", encoding="utf-8") as fh:
        fh.write(cfg_text)
    cfg = lfc.load_config(cfg_path)
    workload = lfc.synthetic_workload(cfg)
    lfc.write_workload(workload.prompts, os.path.join(HERE, "ref_harness_workload.jsonl"))
    report = lfc.run_bench(cfg, workload)
    lfc._write_json(report, os.path.join(HERE, "ref_harness_bench.json"))
    lfc.write_bench_csv(report, os.path.join(HERE, "ref_harness_bench.csv"))
    lfc._write_json(lfc.run_profile(cfg), os.path.join(HERE, "ref_harness_profile.json"))
    code, lines = lfc.run_verify(cfg)
    # perf known answers
    trace = [DispatchEvent("gemm", 2_000_000, 48_000, "backbone"), DispatchEvent("sgmm", 9_000_000, 800_000, "switch"),
             DispatchEvent("gemm", 4_096, 2_048, "router"), DispatchEvent("elementwise", 64, 512, "backbone"),
             DispatchEvent("reduce", 128, 512, "other"), DispatchEvent("gemm", 512, 256, "adapter")]
    cm = lfp.CostModel(2e-6, 5e9, 1e9)
    est = lfp.estimate(trace, cm, n_tokens=3)
    rows = [[r.label, r.kind, r.count, r.flops] for r in lfp.breakdown(trace)]
    samples = [(trace[:2], 0.00231), (trace[:4], 0.00236), (trace, 0.00240), (trace[2:], 0.00009)]
    fit = lfp.calibrate(samples)
    with open(os.path.join(HERE, "ref_perf_expected.json"), "w", encoding="utf-8") as fh:
        json.dump({"trace": [[e.kind, e.flops, e.bytes_touched, e.label] for e in trace],
                   "cost_model": [2e-6, 5e9, 1e9], "n_tokens": 3,
                   "total_ms_per_token": est.total_ms_per_token, "per_component_ms": est.per_component_ms,
                   "dispatch_counts": est.dispatch_counts, "breakdown": rows,
                   "max_compute_fraction": lfp.max_compute_fraction(trace, cm),
                   "calibration_samples": [[len(t), s] for t, s in samples],
                   "calibration_slices": [[0, 2], [0, 4], [0, 6], [2, 6]],
                   "fit_launch_seconds": fit.cost_model.launch_seconds,
                   "fit_flops_throughput": fit.cost_model.flops_throughput,
                   "fit_residuals": [float(r) for r in fit.residuals],
                   "verify_exit_code": code, "verify_lines": lines}, fh, indent=1, sort_keys=True)
    print("harness golden written; reference verify:", code, lines[-1])


if __name__ == "__main__":
    golden_harness()
    golden_io()
    golden_router()
    golden_sgmm()
    golden_switch()
    golden_generate()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)), "bytes")
