"""Time to first token: the batched unmerged prefill (LlamaEngine.prefill) against the step-by-step
merged prompt path, on a workload's full shapes.
    python scripts/bench_prefill.py [workload] [--lengths 16,128,512]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import llama  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload", nargs="?", default="llama2-7b")
ap.add_argument("--lengths", default="16,128,512")
ap.add_argument("--stepwise-max", type=int, default=128)
args = ap.parse_args()
lengths = [int(v) for v in args.lengths.split(",")]
cfg = llama.preset(args.workload, max_seq=max(lengths) + 8)
eng = llama.LlamaEngine(cfg, init="device")
rng = np.random.Generator(np.random.PCG64(3))


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


for T in lengths:
    prompt = [int(t) for t in rng.integers(0, cfg.vocab, T)]
    eng.prefill(prompt)                       # warm-up (cuBLAS handles, allocator)
    ms_b, tok_b = timed(lambda: eng.prefill(prompt))
    line = f"{args.workload} prompt {T:4d}: batched unmerged prefill {ms_b:9.2f} ms ({T / ms_b * 1e3:8.0f} tok/s)"
    if T <= args.stepwise_max:
        def stepwise():
            eng.reset(prompt[0])
            nxt = None
            for t in prompt:
                nxt = eng.decode_step(t)
            return nxt
        ms_s, tok_s = timed(stepwise)
        eng.finalize()
        line += f"; step by step (merged, one switch per token) {ms_s:9.2f} ms ({T / ms_s * 1e3:6.0f} tok/s); same first token: {tok_b == tok_s}"
    print(line, flush=True)
