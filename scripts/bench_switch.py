"""Development benchmark of the fused switch alone on Llama-shaped segment tables.

    python scripts/bench_switch.py [--config 7b|8b|tiny] [--layers L] [--modes mma,fma,exact] [--iters 5]

Prints one JSON line per compute mode: ms per switch, achieved algorithmic GB/s and the
fraction of the measured HBM peak.  Not the contract benchmark (that is bench.py)."""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_11873_b200 as af  # noqa: E402

CONFIGS = {
    "tiny": dict(layers=4, d=256, ffn=0, kv=256, experts=8, rank=8, k=2),
    "7b": dict(layers=32, d=4096, ffn=11008, kv=4096, experts=8, rank=8, k=2),
    "8b": dict(layers=32, d=4096, ffn=14336, kv=1024, experts=16, rank=16, k=2),
    "13b": dict(layers=40, d=5120, ffn=13824, kv=5120, experts=8, rank=8, k=2),
    # one tensor-parallel shard of Llama-2-70B (tp 8): explicit (d_out, d_in) of q k v o gate up down
    "70b-tp8": dict(layers=80, experts=8, rank=32, k=4,
                    shapes=[(1024, 8192), (128, 8192), (128, 8192), (8192, 1024), (3584, 8192), (3584, 8192), (8192, 3584)]),
}


def shapes(c):
    if "shapes" in c:
        return c["shapes"]
    d, ffn, kv = c["d"], c["ffn"], c["kv"]
    if ffn == 0:
        return [(d, d)]
    return [(d, d), (kv, d), (kv, d), (d, d), (ffn, d), (ffn, d), (d, ffn)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="7b")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--modes", default="mma,fma")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--pristine", action="store_true")
    ap.add_argument("--k", type=int, default=0, help="override top-k (stacked ranks of the steady switch = 2 k rank)")
    args = ap.parse_args()
    c = dict(CONFIGS[args.config])
    if args.k:
        c["k"] = args.k
    if args.layers:
        c["layers"] = args.layers
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    targets, downs, ups = [], [], []
    for _ in range(c["layers"]):
        for d_out, d_in in shapes(c):
            w = torch.empty((d_out, d_in), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(d_in ** -0.5)
            targets.append(af.Matrix(w, "bf16"))
            downs.append(torch.empty((c["experts"], c["rank"], d_in), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(d_in ** -0.5))
            ups.append(torch.empty((c["experts"], d_out, c["rank"]), dtype=torch.bfloat16, device=dev).uniform_(-1, 1).mul_(c["rank"] ** -0.5))
    pristine = [t.copy() for t in targets] if args.pristine else None
    table = af.SwitchTable(targets, downs, ups, pristine=pristine)
    info = table.info()
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    rng = np.random.Generator(np.random.PCG64(3))
    k, n_exp = c["k"], c["experts"]

    def decision(disjoint_from=None):
        pool = [e for e in range(n_exp) if disjoint_from is None or e not in disjoint_from]
        ids = tuple(int(v) for v in rng.permutation(pool)[:k])
        w = np.sort(rng.dirichlet(np.ones(k)).astype(np.float32))[::-1]
        return af.GateDecision(ids, tuple(float(v) for v in w))

    print(json.dumps({"config": args.config, "layers": c["layers"], **info, "W_GB": table.target_bytes / 1e9}), flush=True)
    for mode in args.modes.split(","):
        try:
            prev = af.DeviceDecision.from_host(decision())
            table.merge(prev, max_k=k, compute=mode)
            times = []
            for it in range(args.warmup + args.iters):
                cur_h = decision(disjoint_from=prev.to_host().expert_ids)  # worst case: no shared expert, s = 2kr
                cur = af.DeviceDecision.from_host(cur_h)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                table.switch(prev, cur, max_k=k, compute=mode)
                e1.record()
                torch.cuda.synchronize()
                if it >= args.warmup:
                    times.append(e0.elapsed_time(e1))
                prev = cur
            table.status()
            ms = float(np.mean(times))
            s = 2 * k * c["rank"]
            gbs = table.switch_bytes(s) / ms / 1e6
            print(json.dumps({"mode": mode, "kernel": af._capi.lib().af_last_switch_kernel().decode(), "stacked_ranks": s, "ms": round(ms, 4), "min_ms": round(min(times), 4), "GBps": round(gbs, 1),
                              "frac_of_measured_peak": round(gbs / peaks["hbm_gbs"], 4), "bytes": table.switch_bytes(s),
                              "TFLOPs": round(table.switch_flops(s) / ms / 1e9, 1)}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"mode": mode, "error": repr(e)}), flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"# wall {time.time() - t0:.1f}s", flush=True)
