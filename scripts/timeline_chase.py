"""Timeline of the fused switch + GEMV launches of one decode step (af_set_timeline): per launch,
when each CTA entered, had its plan, passed the PDL wait, issued its first/last W load, passed each
phase barrier, finished its prologue / first tile, and when its storer and consumers were done.
Usage: python scripts/timeline_chase.py [workload] [--no-chain] [--layers a,b]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import _capi, llama  # noqa: E402
from paper_2603_11873_b200.linalg import _ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="llama2-7b")
ap.add_argument("--no-chain", action="store_true")
ap.add_argument("--show", default="0,1,2,17,32")
ap.add_argument("--ctx", type=int, default=0, help="positions already in the KV cache")
args = ap.parse_args()

cfg = llama.preset(args.workload, max_seq=args.ctx + 64, forward_mode="chase", chain=not args.no_chain)
eng = llama.LlamaEngine(cfg, init="device")
forced = np.random.Generator(np.random.PCG64(1)).integers(0, cfg.vocab, 64)
eng.reset(forced=forced)
for _ in range(4):
    eng.decode_step(graph=False)
if args.ctx:
    eng.set_position(args.ctx)
SLOTS = 42
n_launch = (cfg.layers + 1) if not args.no_chain else 4 * cfg.layers
grid = _capi.device_info()["sm_count"]
buf = torch.zeros(n_launch * grid * SLOTS, dtype=torch.int64, device="cuda")
_capi.check(_capi.lib().af_set_timeline(_ptr(buf), n_launch, grid * SLOTS))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng._step_body(True)
e1.record()
torch.cuda.synchronize()
_capi.check(_capi.lib().af_set_timeline(None, 0, 0))
print(f"step {e0.elapsed_time(e1):.3f} ms eager, {n_launch} fused launches")
tl = buf.cpu().numpy().reshape(n_launch, grid, SLOTS).astype(np.float64)
smid_all = tl[:, :, 24].copy()
tl[tl == 0] = np.nan
tl[:, :, 24] = smid_all
names = ["entry", "plan", "slab0", "pdlwait", "Wld_first", "Wld_last", "storer_done", "cons_done"]
for ph in range(4):
    names += [f"p{ph}.wait", f"p{ph}.passed", f"p{ph}.prolog", f"p{ph}.tile0"]
t_first = np.nanmin(tl[0, :, 0])
prev_end = None
total_span = 0.0
for i in range(n_launch):
    t0 = np.nanmin(tl[i, :, 0])
    end = np.nanmax(tl[i, :, 6])
    gap = (t0 - prev_end) / 1e3 if prev_end is not None else float("nan")
    total_span += (end - t0) / 1e3
    if str(i) in args.show.split(","):
        print(f"--- launch {i}: starts at {(t0 - t_first) / 1e3:9.1f} us, span {(end - t0) / 1e3:7.1f} us, gap from previous end {gap:6.1f} us")
        for s, nm in enumerate(names):
            col = (tl[i, :, s] - t0) / 1e3
            if np.all(np.isnan(col)):
                continue
            print(f"    {nm:12s} min {np.nanmin(col):7.1f}  med {np.nanmedian(col):7.1f}  max {np.nanmax(col):7.1f} us")
    prev_end = end
if not args.no_chain:
    # per-CTA duration of each phase (barrier passed -> next phase's wait begins), across layers:
    # is a slow CTA always the same SM?
    smid = tl[1, :, 24]
    for ph, nm in ((1, "gate|up"), (2, "down")):
        dur = (tl[1:-1, :, 8 + 4 * (ph + 1)] - tl[1:-1, :, 9 + 4 * ph]) / 1e3      # [launch][cta]
        mean_per_cta = np.nanmean(dur, axis=0)
        order = np.argsort(mean_per_cta)
        print(f"phase {nm}: per-CTA mean duration min {mean_per_cta.min():.1f} med {np.median(mean_per_cta):.1f} max {mean_per_cta.max():.1f} us; "
              f"std across layers (mean over CTAs) {np.nanmean(np.nanstd(dur, axis=0)):.2f} us")
        print("   fastest CTAs (cta:smid:us):", " ".join(f"{c}:{int(smid[c])}:{mean_per_cta[c]:.1f}" for c in order[:10]))
        print("   slowest CTAs (cta:smid:us):", " ".join(f"{c}:{int(smid[c])}:{mean_per_cta[c]:.1f}" for c in order[-10:]))
        same_sm = np.all(tl[1:-1, :, 24] == smid[None, :])
        print("   CTA -> SM mapping identical in every launch:", bool(same_sm))
if not args.no_chain:
    # tcgen05 kernel: the first tile of phase 1 by each epilogue group: loop entry -> operands ready -> chunks done
    for grp in (0, 1):
        a, b, c = (tl[1:-1, :, 26 + 3 * grp + k] for k in range(3))
        pr = tl[1:-1, :, 10 + 4]     # p1.prolog
        if not np.all(np.isnan(a)):
            print(f"phase 1, first tile of epilogue group {grp}: prolog -> loop entry med {np.nanmedian(a - pr) / 1e3:.2f} us, "
                  f"entry -> W tile + accumulator ready med {np.nanmedian(b - a) / 1e3:.2f} us, ready -> four chunks done med {np.nanmedian(c - b) / 1e3:.2f} us")
if not args.no_chain and False:
    # first unit change inside phase 1 (CTAs whose span crosses a strip boundary)
    uc = tl[1:-1, :, 26:32]
    has = ~np.isnan(uc[:, :, 0])
    if has.any():   # (the tcgen05 kernel carries no per-unit stamps)
        d = (uc[:, :, 1:] - uc[:, :, :-1]) / 1e3
        labels = ["wait for all warps", "commit slab + barrier", "new-unit setup", "wait full[stage]", "first tile compute"]
        for k, lb in enumerate(labels):
            v = d[:, :, k][has]
            print(f"unit change: {lb:22s} med {np.nanmedian(v):6.2f}  max {np.nanmax(v):6.2f} us  (n={v.size})")
        fine = tl[1:-1, :, [28, 33, 34, 35, 32, 29]]
        df = (fine[:, :, 1:] - fine[:, :, :-1]) / 1e3
        for k, lb in enumerate(["B fragments (ldmatrix)", "A offsets", "peek + prefetch issue", "x fragment", "ti.next"]):
            v = df[:, :, k][has]
            print(f"   setup: {lb:24s} med {np.nanmedian(v):6.2f}  max {np.nanmax(v):6.2f} us")
# cycles each role spent blocked, as a share of the consumers' lifetime (mean over CTAs and launches)
life = np.nan_to_num(tl[:, :, 41])
ok = life > 0
for slot, nm in () if not ok.any() else ((36, "consumer warp 0 waiting for full[stage] (data)"), (37, "W producer waiting for empty[stage] (ring full)"),
                 (38, "storer waiting for computed[stage]"), (39, "storer waiting for its stores to drain smem")):
    v = np.nan_to_num(tl[:, :, slot])[ok] / life[ok]
    print(f"blocked: {nm:52s} mean {100 * v.mean():5.1f} %  max {100 * v.max():5.1f} %")
t_last = np.nanmax(tl[-1, :, 6])
print(f"first entry -> last storer done: {(t_last - t_first) / 1e3:.1f} us; sum of launch spans {total_span:.1f} us")
