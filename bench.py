"""Contract benchmark of the AdaFuse hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--workload llama2-7b]

A "step" is one decoded token of a bs=1 sequence through the whole hot path: pre-gate on the
token's embedding row, the fused switch of all 7 x L adapted matrices (a teacher-forced token
stream makes every step really switch), the merged-path forward (GQA attention
over the KV cache), lm_head and argmax.  Two schedules of the same arithmetic:
  --forward-mode chase    (default at N=1) each projection's GEMV is fused INTO the switch of its
                          weights: one read + one write of W per token (af_switch_gemv);
  --forward-mode separate ONE switch launch over all matrices, then plain GEMVs (a third pass over W).

  value        tokens/s with every per-step input already in HBM (forced token stream on the
               device, the step replayed as one CUDA graph), max over ranks.
  e2e          the same metric through the public API, verbatim: `eng.decode_step(token)` per step --
               the consumed token goes up from pinned host memory (4 B H2D), the next token and the
               step's status word come back (8 B D2H).
  context      both are timed with `--context` (default 1024) positions already in the KV cache.
  roofline     the fused-switch kernel (chase: its 4 x L launches per token, switch + GEMV):
               algorithmic bytes / launch duration by CUDA events on the launching
               stream -- separate: inside the e2e timed region; chase: in extra e2e steps right
               after it (events between the launches would cut the programmatic overlap the timed
               region runs with) -- against MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline the CPU oracle port (oracle/, reference algorithm restated in C) timed on this
               box's host cores on a bounded sample (whole layers), scaled to tokens/s.

`--impl reference` times that CPU port alone (the reference itself is pure Python and does not
exist on the GPU box): every step is one whole token -- all layers -- when K + W such
steps fit in ~4 minutes, otherwise a bounded sample of layers, and `ms_per_step` is what a step
really took (`value` is then scaled to all layers; `cpu_baseline.sample` says so).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "bs=1 decode tok/s with a fused switch every token (switch us/token and HBM GB/s in extra keys)"
UNIT = "tokens/s"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        return float(json.load(open(path))["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------------ CPU arm ----


_CPU_SEGS: dict = {}


def cpu_sample(cfg_kw: dict, budget_s: float = 15.0, max_layers: int | None = None):
    """Time the oracle port (reference algorithm, f32 arithmetic on bf16 weights) on whole
    layers of the workload: per layer the steady switch of its 7 matrices (s = 2kr) and the 7
    backbone GEMVs.  Returns (seconds per token extrapolated to all layers, layers timed, threads)."""
    from oracle import oracle as orc

    orc.set_num_threads(len(os.sched_getaffinity(0)))   # all host cores, also under torchrun (OMP_NUM_THREADS=1 there)
    d, ffn, L = cfg_kw["hidden"], cfg_kw["ffn"], cfg_kw["layers"]
    hd = d // cfg_kw["n_heads"]
    kv = cfg_kw["n_kv_heads"] * hd
    n, r, k = cfg_kw["experts"], cfg_kw["rank"], cfg_kw["top_k"]
    shapes = [(d, d), (kv, d), (kv, d), (d, d), (ffn, d), (ffn, d), (d, ffn)]
    key = (d, ffn, kv, n, r)
    if _CPU_SEGS.get("key") != key:          # one layer's worth of synthetic matrices, built once (not inside any timed step)
        rng = np.random.Generator(np.random.PCG64(0))
        segs = []
        for d_out, d_in in shapes:
            w = orc.to_bf16_bits((rng.random((d_out, d_in), dtype=np.float32) - 0.5) * (2.0 / np.sqrt(d_in)))
            dn = orc.to_bf16_bits((rng.random((n, r, d_in), dtype=np.float32) - 0.5) * (2.0 / np.sqrt(d_in)))
            up = orc.to_bf16_bits((rng.random((n, d_out, r), dtype=np.float32) - 0.5) * (2.0 / np.sqrt(r)))
            segs.append((w, dn, up, rng.random(d_in, dtype=np.float32)))
        _CPU_SEGS.update(key=key, segs=segs)
    segs = _CPU_SEGS["segs"]
    prev = (tuple(range(k)), tuple([1.0 / k] * k))
    cur = (tuple(range(k, 2 * k)), tuple([1.0 / k] * k))
    done, t_total = 0, 0.0
    cap = max_layers or L
    while done < cap and (done == 0 or t_total + t_total / done <= budget_s):   # at least one layer, then as the budget allows
        t0 = time.perf_counter()
        for w, dn, up, x in segs:
            orc.switch_segment_bf16(w, dn, up, prev, cur)
            orc.gemv_bf16(w, x)
        t_total += time.perf_counter() - t0
        prev, cur = cur, prev
        done += 1
    return t_total / done * L, done, orc.num_threads()


def workload_name(args, cfg_kw) -> str:
    """config.workload — the same string on both arms, so the driver compares like with like."""
    return (f"{args.workload}: Llama-shaped bf16, {cfg_kw['experts']} experts rank {cfg_kw['rank']} top-{cfg_kw['top_k']} "
            f"on q/k/v/o/gate/up/down, bs=1 decode, teacher-forced tokens, switch every token ({args.switch_mode})")


def workload_config(args, cfg_kw, world) -> dict:
    """The `config` object: what is computed, identical on both arms (how it is computed goes to `impl_config`)."""
    return {"workload": workload_name(args, cfg_kw), "parallelism": f"tp{world}", "context_positions": args.context,
            "switch_mode": args.switch_mode, "refresh_every": args.refresh_every,
            "l2": "inputs larger than L2 (weights >= 13 GB >> 126 MB), no flush needed"}


def run_reference_arm(args, cfg_kw):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    L = cfg_kw["layers"]
    # one probe layer sizes the steps: whole tokens when W + K of them fit in ~4 minutes, else a bounded sample of layers
    probe, _, threads = cpu_sample(cfg_kw, budget_s=0.0, max_layers=1)
    n = args.warmup + args.steps
    per_layer = probe / L
    layers_per_step = int(max(1, min(L, 240.0 / max(1, n) / max(per_layer, 1e-9))))
    vals, walls = [], []
    for i in range(n):
        t0 = time.perf_counter()
        sec_per_token, layers_timed, threads = cpu_sample(cfg_kw, budget_s=1e9, max_layers=layers_per_step)
        wall = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(sec_per_token)
            walls.append(wall)
    sec = statistics.mean(vals)
    v = 1.0 / sec
    whole = layers_per_step == L
    sample = (f"every step is one whole token: all {L} layers (steady switch s=2kr + 7 GEMVs each; attention and lm_head not included)"
              if whole else
              f"{layers_per_step} of {L} layers per step (steady switch s=2kr + 7 GEMVs each), value scaled to all layers; "
              f"ms_per_step is the time of the sampled layers")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3, "ms_per_token": sec * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16 storage, f32 accumulate", "data": "synthetic",
        "config": workload_config(args, cfg_kw, args.gpus),
        "impl_config": {"note": "CPU port of the reference algorithm (oracle/liboracle.so, OpenMP, all host cores); "
                                "the reference package itself is pure Python and is not present on the GPU box"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ------------------------------------------------------------------ clocks ----


class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        busy = [c for c in sm if mx and c > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ GPU arm ----


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="llama2-7b")
    ap.add_argument("--switch-mode", default="inplace", choices=["inplace", "from_pristine"])
    ap.add_argument("--compute", default="auto")
    ap.add_argument("--forward-mode", default="auto", choices=["auto", "chase", "separate"])
    ap.add_argument("--no-chain", action="store_true", help="chase: one launch per projection instead of chained phases")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--attn-splits", type=int, default=0, help="KV splits of the decode attention (0 = the engine's choice)")
    ap.add_argument("--persistent-forward", action="store_true",
                    help="plain forward (separate schedule, decode_only) as ONE launch per token (af_forward_persistent) instead of one chained launch per layer")
    ap.add_argument("--context", type=int, default=1024, help="positions already in the KV cache when the timed regions start")
    ap.add_argument("--refresh-every", type=int, default=16,
                    help="in-place mode: rebuild W from the pristine copy every N tokens (reference model.py:344-349; folded into "
                         "that token's switch launch, 0 = never)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    from paper_2603_11873_b200 import llama

    cfg_kw = dict(llama.PRESETS[args.workload])
    if args.impl == "reference":
        run_reference_arm(args, cfg_kw)
        return

    import torch
    import torch.distributed as dist

    from paper_2603_11873_b200 import _capi

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # AF_DIST_BACKEND=gloo with AF_SHARE_DEVICE=1 is the one-GPU rehearsal of the N > 1 path (every rank on cuda:0,
    # collectives staged through the host): it checks the plumbing, its timings mean nothing.
    backend = os.environ.get("AF_DIST_BACKEND", "nccl")
    if os.environ.get("AF_SHARE_DEVICE") == "1":
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    max_seq = args.context + 3 * (args.steps + args.warmup) + 64
    def build_engine(tp_push, peers=None):
        c = llama.preset(args.workload, tp_size=world, tp_rank=rank, max_seq=max_seq, switch_mode=args.switch_mode,
                         compute=args.compute, keep_pristine=True, forward_mode=args.forward_mode, chain=not args.no_chain,
                         attn_splits=args.attn_splits, refresh_every=args.refresh_every, persistent_forward=args.persistent_forward,
                         tp_push=tp_push)
        return c, llama.LlamaEngine(c, init="device", peers=peers)

    # N > 1: the row-parallel sums are pushed into the peers' accumulators from the GEMV epilogue (LlamaConfig.tp_push:
    # torch symmetric memory over NVLink) when the ranks can map each other's buffers -- probed with two eager steps on
    # every rank, all ranks agreeing; otherwise one NCCL all-reduce after o and after down.  AF_TP_PUSH=0 skips the probe.
    tp_collective = "none"
    eng = None
    if world > 1:
        tp_collective = "nccl all-reduce"
        # (AF_TP_PUSH=1 forces the probe on any backend: the one-GPU rehearsal uses it to walk this very code)
        push_env = os.environ.get("AF_TP_PUSH", "auto")
        if (backend == "nccl" or push_env == "1") and push_env != "0" and args.forward_mode != "separate" and not args.no_chain:
            ok = 1
            try:
                try:
                    cfg, eng = build_engine(True)                      # the ranks' buffers in torch symmetric memory
                    tp_how = "torch symmetric memory"
                except RuntimeError:
                    # one node: CUDA IPC handles over the process group instead (also what maps two ranks that share a
                    # GPU, which symmetric memory refuses -- the one-GPU rehearsal)
                    if int(os.environ.get("LOCAL_WORLD_SIZE", "0")) != world:
                        raise
                    dev_ = torch.device("cuda", local_rank)
                    cfg, eng = build_engine(True, peers=lambda n: llama.PeerBuffer.ipc(n, dev_))
                    tp_how = "CUDA IPC"
                eng.reset(forced=[1, 2, 3, 4])
                for _ in range(2):
                    eng.decode_step(graph=False)
                eng.check()
            except Exception as e:   # noqa: BLE001 -- whatever it is, the NCCL path is the fallback
                ok = 0
                print(f"[bench rank {rank}] tp_push unavailable: {type(e).__name__}: {e}", file=sys.stderr, flush=True)
            flag = torch.tensor([ok], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 1:
                tp_collective = f"pushed from the GEMV epilogue (peer memory: {tp_how})"
            else:
                eng = None
                torch.cuda.empty_cache()
    if eng is None:
        cfg, eng = build_engine(False if world > 1 else None)
    info = eng.table.info()
    forced = np.random.Generator(np.random.PCG64(cfg.seed + 1)).integers(0, cfg.vocab, 4096)
    peak, peak_kind = load_peaks()

    def timed(fn, n):
        """n calls of fn bracketed by barrier + synchronize, device time by CUDA events."""
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # ---------------- (1) e2e: the public API verbatim -- eng.decode_step(token): host token in, next token + status out ----
    eng.reset(forced=forced)
    host_tokens = [int(t) for t in forced]
    switch_events = []
    orig_switch = eng._switch_for_step

    def instrumented_switch(with_prev, refresh=False):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        orig_switch(with_prev, refresh)
        b.record()
        switch_events.append((a, b))

    step_i = [0]

    def api_step():
        i = step_i[0]
        eng.decode_step(host_tokens[i % len(host_tokens)])            # 4 B H2D, the whole step, 8 B D2H (token + status word)
        step_i[0] = i + 1

    api_step()                                                         # first merge (no previous decision yet)
    eng.set_position(args.context)                                     # the timed steps attend over >= `context` cached positions
    for _ in range(args.warmup):
        api_step()
    if not eng.chase:
        eng.auto_graph = False          # separate schedule: the timed steps carry events around the switch launch
        eng._switch_for_step = instrumented_switch
    # kernels launched per step, counted on one eagerly launched step (the timed steps replay exactly these as a graph)
    launches0 = _capi.launch_count()
    eng.decode_step(host_tokens[0], graph=False)
    step_launches = _capi.launch_count() - launches0
    sampler = ClockSampler(local_rank)
    profiling = bool(os.environ.get("AF_NCU"))   # `ncu --profile-from-start off`: profile the timed region only
    if profiling:
        torch.cuda.profiler.start()
    e2e_ms = timed(api_step, args.steps)
    if profiling:
        torch.cuda.profiler.stop()
    eng._switch_for_step = orig_switch
    e2e_value = args.steps / (e2e_ms / 1e3)
    chase = eng.chase
    fused_ms = None
    if not chase:
        sw_ms = [a.elapsed_time(b) for a, b in switch_events]
        switch_ms = statistics.mean(sw_ms)
    else:
        # ---- (1b) roofline pass: the same e2e steps with events around every switch + GEMV launch ----
        from paper_2603_11873_b200.adapters import SegmentGroup

        fused_events = []
        orig_sg = SegmentGroup.switch_gemv_chain

        def instrumented_sg(self, *a, **kw):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            orig_sg(self, *a, **kw)
            e1.record()
            fused_events.append((e0, e1))

        SegmentGroup.switch_gemv_chain = instrumented_sg
        eng.auto_graph = False          # eager launches: events around every fused launch
        n_roof = 4
        for _ in range(n_roof):
            api_step()
        torch.cuda.synchronize()
        eng.auto_graph = True
        SegmentGroup.switch_gemv_chain = orig_sg
        per_launch = [a.elapsed_time(b) for a, b in fused_events]
        n_per_step = len(per_launch) // n_roof
        fused_ms = [sum(per_launch[i * n_per_step:(i + 1) * n_per_step]) for i in range(n_roof)]   # per token

    kernel_name = _capi.lib().af_last_switch_kernel().decode()
    # ---------------- (2) value: inputs resident, the step replayed as one CUDA graph ----
    graph_ok = eng.graph_ok()   # one rank, the push step (no library collective inside), or AF_TP_GRAPH=1 (llama.LlamaEngine.graph_ok)
    eng.set_position(args.context)
    if graph_ok:
        eng.capture()
        for _ in range(args.warmup):
            eng.replay()
        dev_ms = timed(eng.replay, args.steps)
        launches_per_step = step_launches
    else:
        def dev_step():
            refresh = eng._refresh_due()
            eng._step_body(not refresh, refresh)
            eng._stepped()
        for _ in range(args.warmup):
            dev_step()
        dev_ms = timed(dev_step, args.steps)
        launches_per_step = step_launches
    clocks = sampler.stop()
    value = args.steps / (dev_ms / 1e3)
    eng.check()

    # ---------------- (3) the adapter-free backbone with the same kernels (decode only) ----
    def decode_only():
        eng.forward()
        eng._advance()

    # (the adapter-free forward of a TP engine still ends its row-parallel GEMVs in library all-reduces: eager unless opted in)
    if world == 1 or os.environ.get("AF_TP_GRAPH") == "1":
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                decode_only()
        torch.cuda.current_stream().wait_stream(side)
        eng.set_position(args.context)
        for _ in range(3):
            g.replay()
        eng.set_position(args.context)
        dec_ms = timed(g.replay, min(args.steps, 30))
        dec_n = min(args.steps, 30)
    else:
        eng.set_position(args.context)
        dec_n = min(args.steps, 30)
        dec_ms = timed(decode_only, dec_n)
    decode_only_tok_s = dec_n / (dec_ms / 1e3)

    # ---------------- (3b) chase: the standalone one-launch switch of the whole table (BASELINE metric
    # "fused-switch us/token"), alternating between two decisions so every launch really switches ----
    if chase:
        from paper_2603_11873_b200.routing import DeviceDecision, GateDecision

        k = cfg.top_k
        da = DeviceDecision.from_host(GateDecision(tuple(range(k)), tuple([1.0 / k] * k)), eng.dev)
        db = DeviceDecision.from_host(GateDecision(tuple(range(k, 2 * k)), tuple([1.0 / k] * k)), eng.dev)
        eng.fused_switch(eng.prev, da)       # live weights now hold decision A
        sw_ms = []
        for i in range(8):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            eng.fused_switch(da if i % 2 == 0 else db, db if i % 2 == 0 else da)
            e1.record()
            torch.cuda.synchronize()
            if i >= 2:
                sw_ms.append(e0.elapsed_time(e1))
        switch_ms = statistics.mean(sw_ms)

    # ---------------- (4) context: this box's own copy bandwidth, measured the way MEASURED_PEAKS.json was
    # (torch b.copy_(a) over 1 Gi bf16 elements, best of 10).  B200s of the pool differ by several per cent.
    box_copy = None
    try:
        a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
        b = torch.empty_like(a)
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        box_copy = 2 * a.numel() * 2 / best / 1e6
        del a, b
    except RuntimeError:
        box_copy = None

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    sw_bytes = cfg.switch_bytes(steady=True)
    achieved = sw_bytes / (switch_ms * 1e-3) / 1e9
    if chase:
        n_launch = n_per_step
        roof_ms = statistics.mean(fused_ms)
        roof_achieved = sw_bytes / (roof_ms * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": kernel_name + " -- fused switch + GEMV; " + ("chained: o -> gate|up -> down -> next q|k|v per launch" if eng.chase_chained else "one launch per projection"),
                    "achieved": roof_achieved, "peak": peak, "unit": "GB/s", "frac": roof_achieved / peak,
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)", "launches_per_token": n_launch,
                    "bytes_per_launch": sw_bytes / n_launch, "avg_launch_ms": roof_ms / n_launch,
                    "bytes_per_token": sw_bytes, "ms_per_token": roof_ms, "min_ms_per_token": min(fused_ms), "traffic": None}
    else:
        roofline = {"bound": "hbm", "kernel": kernel_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                    "bytes_per_launch": sw_bytes, "avg_launch_ms": switch_ms, "min_launch_ms": min(sw_ms), "traffic": None}
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16 storage, f32 accumulate", "data": "synthetic",
        "config": workload_config(args, cfg_kw, world),
        "impl_config": {"segments": info["n_segments"], "work_units": info["n_units"], "compute": args.compute,
                        "forward_mode": "chase (GEMV fused into the switch: W read and written once per token)" if chase
                        else "separate (one switch launch, then plain GEMVs)",
                        "refresh": "every %d-th token switches from the pristine copy (same bytes, same launch)" % eng.refresh_every
                        if eng.refresh_every else "none",
                        "tp_collective": tp_collective},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 4, "d2h_bytes_per_step": 8,
                "ms_per_step": e2e_ms / args.steps,
                "api": "LlamaEngine.decode_step(token): pinned H2D of the token, the step (a CUDA graph replay from the second token on), "
                       "one pinned D2H of next token + status word"},
        "gpu_launches": int(launches_per_step * args.steps),
        "launches_per_step": int(launches_per_step),
        "clocks": clocks,
        "switch_us_per_token": switch_ms * 1e3,
        "switch_hbm_gbs": achieved,
        "decode_only_tok_s": decode_only_tok_s,
        "decode_only_hbm_gbs": cfg.decode_bytes() * decode_only_tok_s / 1e9,
        "decode_only": {"bound": "hbm", "kernel": "gemv_chain_kernel (adapter-free backbone, same attention / lm_head kernels)",
                        "achieved": cfg.decode_bytes() * decode_only_tok_s / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": cfg.decode_bytes() * decode_only_tok_s / 1e9 / peak, "bytes_per_token": cfg.decode_bytes(),
                        "value_over_decode_only": value / decode_only_tok_s,
                        "bound_note": "a token that switches moves every weight twice (read + write back, 2W) where the adapter-free "
                                      "forward reads it once (1W): switch-every-token decode is bounded at %.3f of decode_only by bytes alone; "
                                      "north_star's 'within 10 %% of the adapter-free backbone' is reachable only for steps that keep the "
                                      "previous selection (no bytes written)" % (cfg.decode_bytes() / cfg.switch_bytes(steady=True))},
        "box_hbm_copy_gbs": box_copy,
        "roofline": roofline,
    }
    traffic_path = os.path.join(ROOT, "profiles", "chase_traffic.json" if chase else "switch_traffic.json")
    if os.path.exists(traffic_path):
        try:
            tr = json.load(open(traffic_path))
            if tr.get("workload") == args.workload:
                out["roofline"]["traffic"] = tr.get("dram_bytes_per_launch")
                if chase and tr.get("dram_bytes_per_token"):
                    out["roofline"]["traffic_per_token"] = tr.get("dram_bytes_per_token")
        except (OSError, ValueError):
            pass
    if world > 1:
        out["roofline"]["traffic"] = None   # the ncu capture is of the one-GPU launch, not of a shard's
        out["roofline"].pop("traffic_per_token", None)
    if not args.no_cpu_baseline and world == 1:
        sec_per_token, layers_timed, threads = cpu_sample(cfg_kw, budget_s=15.0)
        out["cpu_baseline"] = {
            "value": 1.0 / sec_per_token, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{layers_timed} of {cfg_kw['layers']} layers (steady switch s=2kr + 7 GEMVs per layer) on the oracle port, "
                      f"scaled to all layers; host has {os.cpu_count()} logical cores",
        }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
