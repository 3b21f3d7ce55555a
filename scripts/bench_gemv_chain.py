"""af_gemv_chain alone: one big phase (steady-state streaming rate) and the four phases of a layer
(o -> gate|up -> down -> q|k|v) back to back, CUDA events around repeated launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import _capi  # noqa: E402

L = _capi.lib()
st = _capi.stream_ptr()
P = _capi.GvPhase
p = lambda t: t.data_ptr()  # noqa: E731


def run(phases, nbytes, label, iters=20):
    arr = (P * len(phases))(*phases)
    done = torch.zeros(4, dtype=torch.int32, device="cuda")
    for _ in range(3):
        done.zero_()
        _capi.check(L.af_gemv_chain(arr, len(phases), p(done), None, 0, st))
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        done.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _capi.check(L.af_gemv_chain(arr, len(phases), p(done), None, 0, st))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{label:44s} {best * 1e3:8.1f} us  {nbytes / best / 1e6:8.1f} GB/s")


d, f = 4096, 11008
mk = lambda r, c: torch.empty((r, c), dtype=torch.bfloat16, device="cuda").uniform_(-0.02, 0.02)  # noqa: E731
x = torch.randn(d, device="cuda")
for rows in (4096, 12288, 22016, 32000, 128000):
    w = mk(rows, d)
    out = torch.zeros(rows, device="cuda")
    run([P(w=p(w), rows=rows, cols=d, ld=d, x=p(x), out=p(out), res=None, norm_w=None, eps=0.0, prologue=0, epilogue=0)], 2 * rows * d,
        f"one phase {rows} x {d}")
wo, wgu, wdn, wq = mk(d, d), mk(2 * f, d), mk(d, f), mk(3 * d, d)
attn, xa, nw = torch.randn(d, device="cuda"), torch.randn(d, device="cuda"), torch.ones(d, device="cuda")
xb, gu, xa2, qkv = torch.zeros(d, device="cuda"), torch.zeros(2 * f, device="cuda"), torch.zeros(d, device="cuda"), torch.zeros(3 * d, device="cuda")
layer = [
    P(w=p(wo), rows=d, cols=d, ld=d, x=p(attn), out=p(xb), res=p(xa), norm_w=None, eps=0.0, prologue=0, epilogue=2),
    P(w=p(wgu), rows=2 * f, cols=d, ld=d, x=p(xb), out=p(gu), res=None, norm_w=p(nw), eps=1e-5, prologue=1, epilogue=0),
    P(w=p(wdn), rows=d, cols=f, ld=f, x=p(gu), out=p(xa2), res=p(xb), norm_w=None, eps=0.0, prologue=2, epilogue=2),
    P(w=p(wq), rows=3 * d, cols=d, ld=d, x=p(xa2), out=p(qkv), res=None, norm_w=p(nw), eps=1e-5, prologue=1, epilogue=0),
]
nb = 2 * (d * d + 2 * f * d + d * f + 3 * d * d)
run(layer, nb, "layer chain o -> gate|up -> down -> q|k|v")
for i, nm in enumerate(("o", "gate|up", "down", "q|k|v")):
    ph = layer[i]
    run([ph], 2 * ph.rows * ph.cols, f"  phase {nm} alone")
