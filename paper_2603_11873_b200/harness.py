"""verify / bench / profile / gen-workload / calibrate, driven by the GPU engine.

The reference's harness (/root/reference/pkg/src/lorafuse/cli.py) prices recorded dispatch traces
with a cost model because it has no device.  This one keeps its file formats -- flat YAML configs
(cli.py:136-163), line-delimited JSON workloads (cli.py:188-226), the schema-1 bench report and its
CSV (cli.py:89-102, 372-420), the profile document (cli.py:507-565), exit codes 0 / 1 / 2
(cli.py:22-23) -- and runs every strategy on the B200, so that next to each *estimated* figure the
report carries the *measured* one (CUDA events around the prefill and the decode loop).  Measured
fields live under ``measured*`` keys and two trailing CSV columns; ``--no-measure`` leaves them out
and the report is then, like the reference's, a pure function of (config, workload, seed).

``calibrate`` (new) closes the loop the reference leaves open (perf.py:167-201): it times
``generate`` on a small grid of shapes and strategies and fits launch cost plus either the flop rate
or the byte bandwidth of the cost model to what the device really did.

Differences a user of the reference will notice: ``precision`` is "bf16" or "single" (no f64 on this
path); ``--workers`` is accepted and ignored (one GPU, prompts run back to back; the report never
depended on it); two extra config keys, ``compute`` and ``switch_mode`` (ModelConfig).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
from dataclasses import dataclass, replace
from datetime import datetime, timezone

import numpy as np

from .errors import CalibrationError, ConfigError, DeviceError, InputError
from .linalg import EVENT_KINDS, DispatchRecorder
from .model import (ModelConfig, Strategy, build_model, decode_step, finalize_generation, generate,
                    max_backbone_deviation, prefill)
from .perf import CostModel, breakdown, calibrate, estimate, measure_samples

SCHEMA_VERSION = 1

STRATEGY_ORDER = (Strategy.BASE, Strategy.LAYER_WISE_ROUTED, Strategy.PRE_GATED_NAIVE,
                  Strategy.PRE_GATED_SIMPLE_MERGE, Strategy.PRE_GATED_FUSED)           # cli.py:54-60
PRE_GATED = tuple(s for s in STRATEGY_ORDER if s.pre_gated)

MODEL_KEYS = ("layers", "hidden", "vocab", "experts", "rank", "top_k", "precision", "seed", "strategy",
              "refresh_every", "compute", "switch_mode")
COST_KEYS = ("launch_seconds", "flops_throughput", "bytes_bandwidth")
WORKLOAD_KEYS = ("n_new", "synthetic_prompts", "synthetic_len_min", "synthetic_len_max")

# max |hidden_a - hidden_b| allowed by verify.  "single" is the reference's figure (cli.py:82-83);
# bf16 weights are re-rounded by every in-place switch, so its bound is the drift bound of
# tests/test_gpu_model.py rather than a round-off bound -- and a drift of that size may flip a greedy
# near-tie, so in bf16 a diverging token stream is reported but only the hidden states (up to and
# including the step where the streams part) are enforced.
VERIFY_TOL = {"single": 1e-3, "bf16": 5e-2}
DEGENERATE_TOL = {"single": 1e-5, "bf16": 5e-2}
TOKENS_ENFORCED = {"single": True, "bf16": False}
RANK_SWEEP = (2, 4, 8, 16)

CSV_COLUMNS = ("schema_version", "strategy", "n_prompts", "n_new", "decode_ms_per_token", "overhead_vs_base_pct",
               "prefill_ms_per_token", "decode_gemm", "decode_sgmm", "decode_elementwise", "decode_reduce",
               "decode_flops")                                                           # cli.py:89-102
CSV_MEASURED_COLUMNS = ("measured_decode_ms_per_token", "measured_prefill_ms_per_token")


@dataclass(frozen=True, slots=True)
class HarnessConfig:
    model: ModelConfig
    cost: CostModel
    n_new: int = 200
    synthetic_prompts: int = 50
    synthetic_len_min: int = 8
    synthetic_len_max: int = 32


@dataclass(frozen=True, slots=True)
class Workload:
    prompts: tuple
    n_new: int

    @property
    def n_prompts(self) -> int:
        return len(self.prompts)

    @property
    def prompt_tokens(self) -> int:
        return sum(map(len, self.prompts))


# ------------------------------------------------------------------ files ----


def load_config(path) -> HarnessConfig:
    """A flat YAML mapping; an unknown key or a bad value is fatal (cli.py:136-163)."""
    import yaml

    try:
        with open(path, "r", encoding="utf-8") as fh:
            doc = yaml.safe_load(fh)
    except yaml.YAMLError as exc:
        raise ConfigError(f"cannot parse config {path}: {exc}") from exc
    doc = {} if doc is None else doc
    if not isinstance(doc, dict):
        raise ConfigError(f"config {path} must be a flat key-value mapping")
    stray = sorted(str(k) for k in doc if k not in MODEL_KEYS + COST_KEYS + WORKLOAD_KEYS)
    if stray:
        raise ConfigError(f"unknown config keys: {', '.join(stray)}")
    if doc.get("precision") == "double":
        raise ConfigError("bad config value: precision 'double' does not exist on the GPU path (use 'single' or 'bf16')")
    try:
        model = ModelConfig.from_dict({k: doc[k] for k in MODEL_KEYS if k in doc})
        cost = CostModel(**{k: float(doc[k]) for k in COST_KEYS if k in doc})
    except (ValueError, TypeError) as exc:
        raise ConfigError(f"bad config value: {exc}") from exc
    shape = {k: doc[k] for k in WORKLOAD_KEYS if k in doc}
    for key, value in shape.items():
        if not isinstance(value, int) or isinstance(value, bool) or value < 1:
            raise ConfigError(f"{key} must be a positive integer, got {value!r}")
    cfg = HarnessConfig(model=model, cost=cost, **shape)
    if cfg.synthetic_len_min > cfg.synthetic_len_max:
        raise ConfigError("synthetic_len_min exceeds synthetic_len_max")
    return cfg


def generate_workload(vocab: int, n_prompts: int, len_min: int, len_max: int, seed: int) -> tuple:
    """Seeded random prompts, the reference's draw order (cli.py:166-178): per prompt one length
    draw from [len_min, len_max], then that many token ids -- so a seed names the same workload in
    both harnesses."""
    if vocab < 2:
        raise ConfigError("vocab must be >= 2")
    if n_prompts < 1 or len_min < 1 or len_max < len_min:
        raise ConfigError("need n_prompts >= 1 and 1 <= len_min <= len_max")
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for _ in range(n_prompts):
        n = int(rng.integers(len_min, len_max + 1))
        out.append(tuple(int(t) for t in rng.integers(0, vocab, size=n)))
    return tuple(out)


def write_workload(prompts, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.writelines(json.dumps({"tokens": list(p)}) + "\n" for p in prompts)


def _prompt_of_record(record, vocab: int, where: str) -> tuple:
    if not isinstance(record, dict):
        raise ConfigError(f"{where}: record must be an object")
    if "tokens" in record:
        ids = record["tokens"]
        if not isinstance(ids, list) or not ids:
            raise ConfigError(f"{where}: tokens must be a non-empty list")
        for t in ids:
            if not isinstance(t, int) or isinstance(t, bool) or not 0 <= t < vocab:
                raise ConfigError(f"{where}: token {t!r} outside vocab of {vocab}")
        return tuple(ids)
    if "text" in record:
        text = record["text"]
        if not isinstance(text, str) or not text:
            raise ConfigError(f"{where}: text must be a non-empty string")
        return tuple(byte % vocab for byte in text.encode("utf-8"))   # byte-level, modulo vocab (cli.py:219-221)
    raise ConfigError(f"{where}: record needs 'tokens' or 'text'")


def load_workload(path, vocab: int, n_new: int) -> Workload:
    """Line-delimited JSON, ``{"tokens": [...]}`` or ``{"text": "..."}`` per line (cli.py:188-226)."""
    prompts = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            raw = raw.strip()
            if not raw:
                continue
            try:
                record = json.loads(raw)
            except json.JSONDecodeError as exc:
                raise ConfigError(f"{path}:{lineno}: not valid JSON: {exc}") from exc
            prompts.append(_prompt_of_record(record, vocab, f"{path}:{lineno}"))
    if not prompts:
        raise ConfigError(f"workload {path} contains no prompts")
    return Workload(tuple(prompts), n_new)


def synthetic_workload(cfg: HarnessConfig) -> Workload:
    m = cfg.model
    return Workload(generate_workload(m.vocab, cfg.synthetic_prompts, cfg.synthetic_len_min, cfg.synthetic_len_max, m.seed),
                    cfg.n_new)


def _timestamp() -> str:
    """ISO-8601 UTC; SOURCE_DATE_EPOCH pins it (cli.py:240-247)."""
    epoch = os.environ.get("SOURCE_DATE_EPOCH")
    when = datetime.fromtimestamp(int(epoch), tz=timezone.utc) if epoch is not None else datetime.now(timezone.utc)
    return when.strftime("%Y-%m-%dT%H:%M:%SZ")


def _config_echo(cfg: HarnessConfig) -> dict:
    echo = cfg.model.to_dict()
    echo.update({k: getattr(cfg.cost, k) for k in COST_KEYS})
    echo.update({k: getattr(cfg, k) for k in WORKLOAD_KEYS})
    return echo


def _device_echo() -> dict:
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("the harness runs the engine on a GPU: no CUDA device is visible")
    props = torch.cuda.get_device_properties(torch.cuda.current_device())
    return {"name": props.name, "sm_count": props.multi_processor_count, "hbm_bytes": props.total_memory}


class _GpuClock:
    """CUDA-event stopwatch on the current stream; ``None`` when measuring is off."""

    def __init__(self, enabled: bool):
        self.enabled = enabled
        if enabled:
            import torch

            self._torch = torch
            self._a, self._b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def start(self) -> None:
        if self.enabled:
            self._torch.cuda.synchronize()
            self._a.record()

    def stop_ms(self):
        if not self.enabled:
            return None
        self._b.record()
        self._torch.cuda.synchronize()
        return float(self._a.elapsed_time(self._b))


# ------------------------------------------------------------------ bench ----


def _bench_one(cfg: HarnessConfig, strategy: Strategy, prompt, n_new: int, measure: bool) -> dict:
    """One (strategy, prompt) pair on a freshly built model (cli.py:270-309): prefill, n_new decode
    steps with the last layer's hidden state kept, restore; the two phases priced separately."""
    model = build_model(replace(cfg.model, strategy=strategy))
    recorder = DispatchRecorder()
    clock = _GpuClock(measure)

    clock.start()
    state = prefill(model, prompt, recorder)
    prefill_ms = clock.stop_ms()
    prefill_events = tuple(recorder.events)

    mark = recorder.mark()
    token, tokens = prompt[-1], []
    final_hidden = np.empty((n_new, cfg.model.hidden))
    clock.start()
    for step in range(n_new):
        layers_out = []
        token, _ = decode_step(model, state, token, recorder, capture=layers_out)
        tokens.append(token)
        final_hidden[step] = layers_out[-1]
    finalize_generation(model, state, recorder)
    decode_ms = clock.stop_ms()
    decode_events = tuple(recorder.events_since(mark))

    pre, dec = estimate(prefill_events, cfg.cost, len(prompt)), estimate(decode_events, cfg.cost, n_new)
    return {
        "tokens": tokens, "final_hidden": final_hidden,
        "prefill_ms_per_token": pre.total_ms_per_token, "prefill_counts": pre.dispatch_counts,
        "decode_ms_per_token": dec.total_ms_per_token, "decode_component_ms": dec.per_component_ms,
        "decode_counts": dec.dispatch_counts, "decode_flops": sum(ev.flops for ev in decode_events),
        "restore_dev": max_backbone_deviation(model),
        "measured_prefill_ms": prefill_ms, "measured_decode_ms": decode_ms,
    }


def run_bench(cfg: HarnessConfig, workload: Workload, workers: int = 1, measure: bool = True) -> dict:
    """All five strategies over the workload -> the schema-1 report (cli.py:312-392), plus measured
    ms/token per strategy when ``measure``."""
    del workers  # one GPU: prompts run back to back; the report never depended on the worker count
    device = _device_echo()
    runs = {s: [_bench_one(cfg, s, p, workload.n_new, measure) for p in workload.prompts] for s in STRATEGY_ORDER}
    n = workload.n_prompts
    summaries = {}
    for strat, rows in runs.items():
        summary = {
            "decode_ms_per_token": sum(r["decode_ms_per_token"] for r in rows) / n,
            "per_prompt_decode_ms": [r["decode_ms_per_token"] for r in rows],
            "per_component_ms": {label: sum(r["decode_component_ms"][label] for r in rows) / n
                                 for label in rows[0]["decode_component_ms"]},
            "dispatch_counts_decode": {k: sum(r["decode_counts"][k] for r in rows) for k in EVENT_KINDS},
            "dispatch_counts_prefill": {k: sum(r["prefill_counts"][k] for r in rows) for k in EVENT_KINDS},
            "decode_flops": sum(r["decode_flops"] for r in rows),
            # token-weighted, as the reference does it (cli.py:336-338)
            "prefill_ms_per_token": sum(r["prefill_ms_per_token"] * len(p) for r, p in zip(rows, workload.prompts))
                                    / workload.prompt_tokens,
            "max_backbone_restore_dev": max(r["restore_dev"] for r in rows),
            "tokens_digest": hashlib.sha256(json.dumps([r["tokens"] for r in rows]).encode("utf-8")).hexdigest(),
        }
        if measure:
            summary["measured_decode_ms_per_token"] = sum(r["measured_decode_ms"] for r in rows) / (n * workload.n_new)
            summary["measured_prefill_ms_per_token"] = sum(r["measured_prefill_ms"] for r in rows) / workload.prompt_tokens
        summaries[strat] = summary
    base = summaries[Strategy.BASE]
    for summary in summaries.values():
        summary["overhead_vs_base_pct"] = 100.0 * (summary["decode_ms_per_token"] - base["decode_ms_per_token"]) \
            / base["decode_ms_per_token"]
        if measure:
            summary["measured_overhead_vs_base_pct"] = 100.0 * (
                summary["measured_decode_ms_per_token"] - base["measured_decode_ms_per_token"]) / base["measured_decode_ms_per_token"]

    # reported, not enforced -- verify is the enforcing command (cli.py:355-374)
    pairs, all_match = {}, True
    for i, a in enumerate(PRE_GATED):
        for b in PRE_GATED[i + 1:]:
            same = all(ra["tokens"] == rb["tokens"] for ra, rb in zip(runs[a], runs[b]))
            dev = max(float(np.max(np.abs(ra["final_hidden"] - rb["final_hidden"]))) for ra, rb in zip(runs[a], runs[b]))
            pairs[f"{a.value}|{b.value}"] = {"max_final_hidden_dev": dev, "tokens_match": same}
            all_match = all_match and same
    report = {
        "schema_version": SCHEMA_VERSION, "kind": "bench", "timestamp": _timestamp(), "seed": cfg.model.seed,
        "config": _config_echo(cfg),
        "workload": {"n_prompts": n, "n_new": workload.n_new, "prompt_tokens": workload.prompt_tokens},
        "strategies": {s.value: summaries[s] for s in STRATEGY_ORDER},
        "equivalence": {"tokens_match": all_match, "pairs": pairs},
    }
    if measure:
        report["measured"] = {"device": device, "clock": "CUDA events around prefill and around the decode loop "
                                                         "(restore included), per prompt, summed"}
    return report


def write_json(doc, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def csv_path(out_path: str) -> str:
    return os.path.splitext(out_path)[0] + ".csv"


def write_bench_csv(report: dict, path) -> None:
    """One row per strategy, the reference's columns first (cli.py:395-420); measured columns are
    appended only when the report has them."""
    measured = "measured" in report
    header = CSV_COLUMNS + (CSV_MEASURED_COLUMNS if measured else ())
    lines = [",".join(header)]
    for strat in STRATEGY_ORDER:
        s = report["strategies"][strat.value]
        c = s["dispatch_counts_decode"]
        row = [str(report["schema_version"]), strat.value, str(report["workload"]["n_prompts"]),
               str(report["workload"]["n_new"]), repr(float(s["decode_ms_per_token"])),
               repr(float(s["overhead_vs_base_pct"])), repr(float(s["prefill_ms_per_token"])), str(c["gemm"]),
               str(c["sgmm"]), str(c["elementwise"]), str(c["reduce"]), str(s["decode_flops"])]
        if measured:
            row += [repr(float(s[k])) for k in CSV_MEASURED_COLUMNS]
        lines.append(",".join(row))
    with open(path, "w", encoding="utf-8", newline="\n") as fh:
        fh.write("\n".join(lines) + "\n")


# ----------------------------------------------------------------- verify ----


def _hidden_dev(tokens_a, hid_a, tokens_b, hid_b) -> float:
    """max |a - b| over the steps both runs computed from the same consumed tokens: every step up to
    and including the first one whose *emitted* token differs (later steps consume different tokens
    and are incomparable)."""
    worst = 0.0
    for ta, ha, tb, hb in zip(tokens_a, hid_a, tokens_b, hid_b):
        same = next((i for i, (x, y) in enumerate(zip(ta, tb)) if x != y), len(ta) - 1) + 1
        worst = max(worst, float(np.max(np.abs(ha[:same] - hb[:same]))))
    return worst


def run_verify(cfg: HarnessConfig):
    """Pre-gated strategies must agree on a seeded prompt set (cli.py:428-487): 4 prompts of 6
    tokens, min(n_new, 32) steps, every layer of every step.  Token streams must be identical
    (precision "single") and hidden states within VERIFY_TOL; with experts = top_k = 1 the layer-wise strategy is held to the
    naive one too.  Returns (exit code, lines)."""
    _device_echo()
    precision = cfg.model.precision
    tol = VERIFY_TOL[precision]
    strict = TOKENS_ENFORCED[precision]
    differ = "DIFFER" if strict else "differ (near-tie flip under bf16 drift; not enforced)"
    rng = np.random.Generator(np.random.PCG64(cfg.model.seed))
    prompts = [tuple(int(t) for t in rng.integers(0, cfg.model.vocab, size=6)) for _ in range(4)]
    n_new = min(cfg.n_new, 32)

    def run(strategy: Strategy):
        model = build_model(replace(cfg.model, strategy=strategy))
        streams, hiddens = [], []
        for prompt in prompts:
            sink = []
            out, _ = generate(model, prompt, n_new, DispatchRecorder(), hidden_sink=sink)
            streams.append(out)
            hiddens.append(np.array([np.stack(step) for step in sink]))
        return streams, hiddens

    got = {s: run(s) for s in PRE_GATED}
    lines, ok = [], True
    for i, a in enumerate(PRE_GATED):
        for b in PRE_GATED[i + 1:]:
            dev = _hidden_dev(*got[a], *got[b])
            same = got[a][0] == got[b][0]
            ok = ok and (same or not strict) and dev <= tol
            lines.append(f"{a.value} ~ {b.value}: max hidden deviation {dev:.3e} (tolerance {tol:.0e}), "
                         f"tokens {'identical' if same else differ}")
    if cfg.model.experts == 1 and cfg.model.top_k == 1:
        dtol = DEGENERATE_TOL[precision]
        lw = run(Strategy.LAYER_WISE_ROUTED)
        naive = got[Strategy.PRE_GATED_NAIVE]
        dev, same = _hidden_dev(*lw, *naive), lw[0] == naive[0]
        ok = ok and (same or not strict) and dev <= dtol
        lines.append(f"layer_wise_routed ~ pre_gated_naive (experts=1, top_k=1): max hidden deviation {dev:.3e} "
                     f"(tolerance {dtol:.0e}), tokens {'identical' if same else differ}")
    lines.append("verify: " + ("PASS" if ok else "FAIL"))
    return (0 if ok else 1), lines


# ---------------------------------------------------------------- profile ----


def _steady_step(model, warm_token: int, measure: bool):
    """Events (and measured ms) of one steady decode step: a one-token prefill, one warm step, then
    the step that is reported (cli.py:495-502)."""
    recorder = DispatchRecorder()
    state = prefill(model, (warm_token,), recorder)
    token, _ = decode_step(model, state, warm_token, recorder)
    clock = _GpuClock(measure)
    mark = recorder.mark()
    clock.start()
    decode_step(model, state, token, recorder)
    ms = clock.stop_ms()
    return tuple(recorder.events_since(mark)), ms


def _section(events, cost: CostModel, n_tokens: int, measured_ms) -> dict:
    est = estimate(events, cost, n_tokens)
    out = {"rows": [[r.label, r.kind, r.count, r.flops] for r in breakdown(events)],
           "ms_per_token": est.total_ms_per_token, "per_component_ms": est.per_component_ms,
           "dispatch_counts": est.dispatch_counts}
    if measured_ms is not None:
        out["measured_ms_per_token"] = measured_ms / n_tokens
    return out


def run_profile(cfg: HarnessConfig, measure: bool = True) -> dict:
    """Per-component breakdown of one steady decode step and of a 100-token prefill for every
    strategy, and the adapter-rank sweep on the layer-wise strategy (cli.py:507-565)."""
    device = _device_echo()
    rng = np.random.Generator(np.random.PCG64(cfg.model.seed))
    warm_token = int(rng.integers(0, cfg.model.vocab))
    long_prompt = tuple(int(t) for t in rng.integers(0, cfg.model.vocab, size=100))
    decode_section, prefill_section = {}, {}
    for strat in STRATEGY_ORDER:
        events, ms = _steady_step(build_model(replace(cfg.model, strategy=strat)), warm_token, measure)
        decode_section[strat.value] = _section(events, cfg.cost, 1, ms)
        model = build_model(replace(cfg.model, strategy=strat))
        recorder, clock = DispatchRecorder(), _GpuClock(measure)
        clock.start()
        prefill(model, long_prompt, recorder)
        ms = clock.stop_ms()
        prefill_section[strat.value] = _section(tuple(recorder.events), cfg.cost, len(long_prompt), ms)
    sweep = {"rank": [], "adapter_ms_per_token": [], "adapter_flops_per_token": []}
    if measure:
        sweep["measured_ms_per_token"] = []
    for rank in RANK_SWEEP:
        if rank > cfg.model.hidden:
            continue
        model = build_model(replace(cfg.model, rank=rank, strategy=Strategy.LAYER_WISE_ROUTED))
        events, ms = _steady_step(model, warm_token, measure)
        sweep["rank"].append(rank)
        sweep["adapter_ms_per_token"].append(estimate(events, cfg.cost, 1).per_component_ms["adapter"])
        sweep["adapter_flops_per_token"].append(sum(ev.flops for ev in events if ev.label == "adapter"))
        if measure:
            sweep["measured_ms_per_token"].append(ms)
    doc = {"schema_version": SCHEMA_VERSION, "kind": "profile", "timestamp": _timestamp(), "seed": cfg.model.seed,
           "config": _config_echo(cfg), "decode_step": decode_section, "prefill_100": prefill_section, "rank_sweep": sweep}
    if measure:
        doc["measured"] = {"device": device, "clock": "CUDA events around the reported step / the prefill"}
    return doc


# -------------------------------------------------------------- calibrate ----


def run_calibrate(cfg: HarnessConfig, n_new: int = 16) -> dict:
    """Fit the cost model to this device: ``generate`` timed on {hidden, 2 hidden, 4 hidden} x
    {base, fused} (six different events-to-work mixes), then perf.calibrate with the reference's
    flop regressor and with the byte regressor; each fit reports its residuals, or why it failed."""
    device = _device_echo()
    grid = [replace(cfg.model, hidden=cfg.model.hidden * mult, strategy=strat)
            for mult in (1, 2, 4) for strat in (Strategy.BASE, Strategy.PRE_GATED_FUSED)]
    pairs = measure_samples(grid, n_new=n_new)
    doc = {"schema_version": SCHEMA_VERSION, "kind": "calibration", "timestamp": _timestamp(), "seed": cfg.model.seed,
           "config": _config_echo(cfg), "device": device,
           "samples": [{"hidden": g.hidden, "strategy": g.strategy.value, "n_events": len(trace),
                        "flops": sum(ev.flops for ev in trace), "bytes": sum(ev.bytes_touched for ev in trace),
                        "seconds": secs} for g, (trace, secs) in zip(grid, pairs)],
           "fits": {}}
    for regressor in ("flops", "bytes"):
        try:
            fit = calibrate(pairs, regressor=regressor)
            doc["fits"][regressor] = {"launch_seconds": fit.cost_model.launch_seconds,
                                      "flops_throughput": fit.cost_model.flops_throughput,
                                      "bytes_bandwidth": fit.cost_model.bytes_bandwidth,
                                      "residual_seconds": [float(r) for r in fit.residuals]}
        except CalibrationError as exc:
            doc["fits"][regressor] = {"error": str(exc)}
    return doc


# ------------------------------------------------------------------- main ----


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="adafuse-b200", description="verify / bench / profile the pre-gated LoRA decoder "
                                 "on the GPU engine; file formats of the reference harness")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("verify", help="check that the pre-gated strategies agree")
    p.add_argument("--config", required=True)
    p = sub.add_parser("bench", help="estimated and measured per-strategy decode latency")
    p.add_argument("--config", required=True)
    src = p.add_mutually_exclusive_group(required=True)
    src.add_argument("--workload", help="line-delimited JSON workload file")
    src.add_argument("--synthetic", action="store_true", help="the seeded synthetic workload of the config")
    p.add_argument("--out", required=True, help="JSON report path; the CSV is written beside it")
    p.add_argument("--workers", type=int, default=1, help="accepted for compatibility; one GPU runs the prompts in order")
    p.add_argument("--no-measure", action="store_true", help="leave the measured fields out (reproducible report)")
    p = sub.add_parser("profile", help="per-component dispatch breakdowns")
    p.add_argument("--config", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--no-measure", action="store_true")
    p = sub.add_parser("gen-workload", help="write a random token-id workload")
    p.add_argument("--vocab", type=int, required=True)
    p.add_argument("--prompts", type=int, required=True)
    p.add_argument("--len", dest="len_range", required=True, metavar="MIN:MAX")
    p.add_argument("--seed", type=int, required=True)
    p.add_argument("--out", required=True)
    p = sub.add_parser("calibrate", help="fit the cost model to times measured on this GPU")
    p.add_argument("--config", required=True)
    p.add_argument("--out", required=True)
    return ap


def _len_range(text: str):
    lo, sep, hi = text.partition(":")
    try:
        if not sep:
            raise ValueError(text)
        return int(lo), int(hi)
    except ValueError as exc:
        raise ConfigError(f"--len must look like MIN:MAX, got {text!r}") from exc


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    try:
        if args.command == "gen-workload":
            lo, hi = _len_range(args.len_range)
            prompts = generate_workload(args.vocab, args.prompts, lo, hi, args.seed)
            write_workload(prompts, args.out)
            print(f"wrote {len(prompts)} prompts to {args.out}")
            return 0
        cfg = load_config(args.config)
        if args.command == "verify":
            code, lines = run_verify(cfg)
            print("\n".join(lines))
            return code
        if args.command == "bench":
            if args.workers < 1:
                raise ConfigError("--workers must be >= 1")
            workload = synthetic_workload(cfg) if args.synthetic else load_workload(args.workload, cfg.model.vocab, cfg.n_new)
            report = run_bench(cfg, workload, workers=args.workers, measure=not args.no_measure)
            write_json(report, args.out)
            write_bench_csv(report, csv_path(args.out))
            print(f"wrote {args.out} and {csv_path(args.out)}")
            return 0
        if args.command == "profile":
            write_json(run_profile(cfg, measure=not args.no_measure), args.out)
            print(f"wrote {args.out}")
            return 0
        if args.command == "calibrate":
            write_json(run_calibrate(cfg), args.out)
            print(f"wrote {args.out}")
            return 0
    except (ConfigError, InputError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except DeviceError as exc:
        print(f"device error: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"i/o error: {exc}", file=sys.stderr)
        return 2
    raise AssertionError("unreachable")


if __name__ == "__main__":  # pragma: no cover
    sys.exit(main())
