"""BASELINE.json configs[2]: switch-every-token vs cached-selection sweep.

For switch period P in {1, 2, 4, 8, 16, inf} the routing decision is refreshed (pre-gate + fused
switch) every P-th token and held in between (hold steps run the merged forward only).  P > 1
changes the outputs (a held selection is not the reference's per-token routing), so parity is a
P = 1 statement; this script reports throughput only.

    python scripts/bench_sweep.py [llama3-8b] [--steps 48] [--switch-mode inplace|from_pristine]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import llama  # noqa: E402


def capture(fn):
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload", nargs="?", default="llama3-8b")
    ap.add_argument("--steps", type=int, default=48)
    ap.add_argument("--switch-mode", default="inplace")
    ap.add_argument("--forward-mode", default="auto", choices=["auto", "chase", "separate"])
    ap.add_argument("--context", type=int, default=1024, help="positions already in the KV cache")
    args = ap.parse_args()
    # (refresh_every = 0: the sweep's graphs are captured by hand; the refreshing step costs the same as a steady one)
    cfg = llama.preset(args.workload, max_seq=args.context + 8 * args.steps + 64, switch_mode=args.switch_mode, forward_mode=args.forward_mode,
                       refresh_every=0)
    eng = llama.LlamaEngine(cfg, init="device")
    forced = np.random.Generator(np.random.PCG64(7)).integers(0, cfg.vocab, 4096)
    eng.reset(forced=forced)
    for _ in range(3):
        eng.decode_step(graph=False)
    g_switch = capture(lambda: eng._step_body(True))

    def hold():
        eng.forward()
        eng._advance()

    g_hold = capture(hold)
    peak = 6554.9
    try:
        peak = float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
    except OSError:
        pass
    lm_head_bytes = 2 * (cfg.vocab // cfg.tp_size) * cfg.hidden
    # a switching step moves the switch bytes and, in the separate schedule, the forward's bytes on top;
    # in the chase schedule the forward rides on the switch's pass (only lm_head is extra)
    switch_step_bytes = cfg.switch_bytes() + (lm_head_bytes if eng.chase else cfg.decode_bytes())
    print(json.dumps({"workload": args.workload, "context_positions": args.context, "switch_mode": args.switch_mode, "forward_mode": "chase" if eng.chase else "separate",
                      "segments": eng.table.info()["n_segments"],
                      "switch_bytes": cfg.switch_bytes(), "decode_bytes": cfg.decode_bytes()}), flush=True)
    for period in (1, 2, 4, 8, 16, 0):
        eng.set_position(args.context)
        for _ in range(2):
            g_switch.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n_sw = 0
        for i in range(args.steps):
            if period and i % period == 0:
                g_switch.replay()
                n_sw += 1
            else:
                g_hold.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        bytes_per_tok = (switch_step_bytes * n_sw + cfg.decode_bytes() * (args.steps - n_sw)) / args.steps
        print(json.dumps({"switch_period": period if period else "inf", "switches": n_sw, "ms_per_token": round(ms, 4),
                          "tok_s": round(1e3 / ms, 1), "hbm_GBps": round(bytes_per_tok / ms / 1e6, 1),
                          "frac_of_measured_peak": round(bytes_per_tok / ms / 1e6 / peak, 4)}), flush=True)
    eng.check()


if __name__ == "__main__":
    main()
