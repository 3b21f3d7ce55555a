"""Per-GPU decode step of ONE tensor-parallel shard, timed alone on one GPU (no peers: the collectives
are no-ops, so this is the compute + HBM time a rank spends per token, without NCCL latency).
    python scripts/bench_shard.py llama2-13b --tp 2 [--steps 30] [--forward-mode auto|chase|separate]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import llama  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="llama2-13b")
ap.add_argument("--tp", type=int, default=2)
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--forward-mode", default="auto")
ap.add_argument("--switch-mode", default="inplace")
ap.add_argument("--push", action="store_true", help="tp_push step (chained launches, sums pushed from the epilogue) with the rank as its only peer")
args = ap.parse_args()


class Alone(llama.Collectives):
    def __init__(self, tp):
        self.group, self.tp_size = None, tp

    def all_reduce_sum(self, t):
        pass

    def broadcast_decision(self, buf):
        pass

    def argmax_pairs(self, val, idx, out_idx):
        pass


cfg = llama.preset(args.workload, tp_size=args.tp, tp_rank=0, max_seq=2 * args.steps + 32, forward_mode=args.forward_mode,
                   switch_mode=args.switch_mode, tp_push=True if args.push else False)
dev = torch.device("cuda", 0)
eng = llama.LlamaEngine(cfg, init="device", comm=Alone(args.tp), peers=(lambda n: llama.PeerBuffer.local(n, dev)) if args.push else None)
forced = np.random.Generator(np.random.PCG64(1)).integers(0, cfg.vocab, 256)
eng.reset(forced=forced)
for _ in range(4):
    eng.decode_step()


def timed(fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


eager = timed(lambda: eng._step_body(True), args.steps)
# the same step as a CUDA graph (what a rank's step costs once the host launches are out of the way)
g = torch.cuda.CUDAGraph()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    with torch.cuda.graph(g, stream=side):
        eng._step_body(True)
torch.cuda.current_stream().wait_stream(side)
for _ in range(3):
    g.replay()
graph = timed(g.replay, args.steps)
info = eng.table.info()
w_gb = sum(t.data.numel() for t in eng.targets) * 2 / 1e9
print(f"{args.workload} tp{args.tp} rank 0 alone: W {w_gb:.2f} GB/rank, stacked ranks {2 * cfg.top_k * cfg.rank}, "
      f"schedule {'chase' if eng.chase else 'separate'}{' chained + push (alone)' if getattr(eng, 'tp_push', False) else ''}, tensor path {bool(info.get('tensor_path'))}, tcgen05 {bool(info.get('umma_path'))}: "
      f"eager {eager:.3f} ms/token, graph {graph:.3f} ms/token ({1e3 / graph:.0f} tok/s per rank-step; "
      f"{(3 if not eng.chase else 2) * w_gb / graph * 1e3:.0f} GB/s of W traffic at 2 (chase) / 3 (separate) passes over W)", flush=True)
