"""Development benchmark: adapter-free decode forward (the merged-path GEMV chain) as one CUDA
graph, for every GEMV streaming variant x PDL on/off.  Prints tokens/s and achieved HBM GB/s."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_11873_b200 import _capi, llama  # noqa: E402


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "llama2-7b"
    chain = os.environ.get("AF_GEMV_CHAIN", "1") != "0"   # one persistent launch per layer (af_gemv_chain) vs one launch per projection
    cfg = llama.preset(workload, max_seq=256, adapters=False, gemv_chain=chain)
    eng = llama.LlamaEngine(cfg, init="device")
    L = _capi.lib()
    combos = ((0, 0), (1, 0), (2, 0), (3, 0), (4, 0), (2, 1), (4, 1), (3, 1))
    if len(sys.argv) > 2:
        combos = tuple((int(v), 0) for v in sys.argv[2].split(","))
    for variant, full_sm in combos:
        for pdl in (1, 0):
            _capi.check(L.af_set_gemv_variant(variant, full_sm))
            _capi.check(L.af_set_pdl(pdl))
            eng.reset(0)
            for _ in range(3):
                eng.forward(); eng._advance()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    eng.forward(); eng._advance()
            torch.cuda.current_stream().wait_stream(side)
            for _ in range(3):
                g.replay()
            eng.pos_dev.fill_(8)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            n = 30
            e0.record()
            for _ in range(n):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / n
            print(json.dumps({"chain": chain, "variant": variant, "full_sm": full_sm, "pdl": pdl, "ms_per_token": round(ms, 4),
                              "tok_s": round(1e3 / ms, 1), "GBps": round(cfg.decode_bytes() / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
