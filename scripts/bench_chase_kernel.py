"""Steady-state rate of the fused switch + GEMV kernel on one projection group, without the
decode chain around it: `n` layers of a workload's shapes, the same group of every layer launched
back to back (no dependencies between them), CUDA events around the whole sequence.
    python scripts/bench_chase_kernel.py [workload] [--layers 8] [--group gu|qkv|o|down]
Env: AF_UMMA=0 selects the mma.sync kernel; AF_DBG=4 runs the plain switch kernel on the group's schedule
(mma.sync path), AF_DBG=8 / 16 / 24 switch the L2 evict-first hints of the W loads / stores off."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import llama  # noqa: E402
from paper_2603_11873_b200.adapters import SegmentGroup  # noqa: E402
from paper_2603_11873_b200.routing import DeviceDecision, GateDecision  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="llama2-7b")
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--plain", action="store_true", help="no decisions: the launch is a plain GEMV (reads W once, stores nothing)")
args = ap.parse_args()
cfg = llama.preset(args.workload, layers=args.layers, max_seq=16, forward_mode="separate", keep_pristine=False)
eng = llama.LlamaEngine(cfg, init="device")
k = cfg.top_k
da = DeviceDecision.from_host(GateDecision(tuple(range(k)), tuple([1.0 / k] * k)), eng.dev)
db = DeviceDecision.from_host(GateDecision(tuple(range(k, 2 * k)), tuple([1.0 / k] * k)), eng.dev)
eng.fused_switch(None, da)
shp = cfg.segment_shapes()
s = 2 * k * cfg.rank
ids = {"qkv": [0, 1, 2], "o": [3], "gu": [4, 5], "down": [6]}
names = {"qkv": ["q", "k", "v"], "o": ["o"], "gu": ["gate", "up"], "down": ["down"]}
for gname in ("gu", "qkv", "down", "o"):
    groups = [SegmentGroup(eng.table, [7 * li + j for j in ids[gname]]) for li in range(cfg.layers)]
    nbytes = sum(4 * shp[n][0] * shp[n][1] + 2 * s * (shp[n][0] + shp[n][1]) for n in names[gname])
    if args.plain:
        nbytes = sum(2 * shp[n][0] * shp[n][1] for n in names[gname])
    x = torch.randn(groups[0].x_len, device="cuda")
    acc = torch.zeros(groups[0].y_rows, dtype=torch.int64, device="cuda")
    best = 1e9
    for it in range(args.iters):
        prev, cur = (da, db) if it % 2 == 0 else (db, da)
        if args.plain:
            prev = cur = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for g in groups:
            g.switch_gemv(prev, cur, acc, xin=x, max_k=k)
        e1.record()
        torch.cuda.synchronize()
        if it >= 2:
            best = min(best, e0.elapsed_time(e1))
    us = best * 1e3 / cfg.layers
    print(f"AF_DBG={os.environ.get('AF_DBG', '0')}{' plain-GEMV' if args.plain else ''} group {gname:4s}: {us:7.1f} us per launch, {nbytes / us / 1e3:7.1f} GB/s ({groups[0].tiles} tiles, grid {groups[0].grid})")
