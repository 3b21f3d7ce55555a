"""Soak: many replays of the captured chase step (in-kernel phase barriers, fixed-point atomics) --
no device-side timeout flag, deterministic tokens across two identical runs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import llama  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
runs = []
for rep in range(2):
    cfg = llama.preset("llama2-7b", max_seq=n + 16)
    eng = llama.LlamaEngine(cfg, init="device")
    forced = np.random.Generator(np.random.PCG64(3)).integers(0, cfg.vocab, 4096)
    eng.reset(forced=forced)
    eng.decode_step()
    eng.capture()
    for _ in range(n):
        eng.replay()
    torch.cuda.synchronize()
    eng.check()          # the engine's status word: unusable decision / phase-barrier timeout
    runs.append(eng.tokens())
    del eng
    torch.cuda.empty_cache()
print("steps", len(runs[0]), "identical across runs:", runs[0] == runs[1], "distinct tokens:", len(set(runs[0])))
assert runs[0] == runs[1]
