"""Decode attention alone (af_attn_decode_fix) at a given context length: us per launch as a function of the KV split count.
    python scripts/bench_attn.py [--ctx 1024] [--heads 32] [--kv 32] [--hd 128]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import _capi  # noqa: E402
from paper_2603_11873_b200.linalg import _ptr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, default=1024)
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv", type=int, default=32)
ap.add_argument("--hd", type=int, default=128)
ap.add_argument("--splits", default="1,2,4,8,12,16,24,32")
args = ap.parse_args()
L, st = _capi.lib(), None
dev = torch.device("cuda")
nh, nkv, hd = args.heads, args.kv, args.hd
max_seq = args.ctx + 64
n_layers = 8            # distinct caches so that consecutive launches do not hit L2 on the same KV
kc = [torch.randn(nkv, max_seq, hd, device=dev).to(torch.bfloat16) for _ in range(n_layers)]
vc = [torch.randn(nkv, max_seq, hd, device=dev).to(torch.bfloat16) for _ in range(n_layers)]
qkv = (torch.randn((nh + 2 * nkv) * hd, device=dev) * 2 ** 40).to(torch.int64)
cos = torch.rand(max_seq, hd // 2, device=dev)
sin = torch.rand(max_seq, hd // 2, device=dev)
pos = torch.full((1,), args.ctx, dtype=torch.int32, device=dev)
out = torch.zeros(nh * hd, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for splits in [int(s) for s in args.splits.split(",")]:
    ws = torch.zeros(nh * splits * (hd + 2), device=dev)
    tickets = torch.zeros(nh, dtype=torch.int32, device=dev)

    def launch(i):
        _capi.check(L.af_attn_decode_fix(_ptr(qkv), None, _ptr(kc[i % n_layers]), _ptr(vc[i % n_layers]), _ptr(cos), _ptr(sin), _ptr(pos),
                                         nh, nkv, hd, max_seq, splits, _ptr(ws), _ptr(tickets), _ptr(out), _capi.stream_ptr()))

    for i in range(4):
        launch(i)
    torch.cuda.synchronize()
    times = []
    for rep in range(5):
        flush.zero_()                       # KV out of L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(n_layers):
            launch(i)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / n_layers * 1e3)
    kv_mb = 2 * nkv * args.ctx * hd * 2 / 1e6
    print(f"ctx {args.ctx} heads {nh}/{nkv} hd {hd} splits {splits:2d}: {min(times):6.2f} us / launch (KV {kv_mb:.1f} MB -> {kv_mb / min(times) * 1e3:.0f} GB/s)", flush=True)
