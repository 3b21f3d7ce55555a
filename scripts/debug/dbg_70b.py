"""Locate where a Llama-2-70B tp8 shard's switch leaves the oracle (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from oracle import oracle as orc
from paper_2603_11873_b200 import llama

def bits(t):
    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16).copy()

for mode in sys.argv[1:] or ["separate", "chase"]:
    cfg = llama.preset("llama2-70b", tp_size=8, tp_rank=0, layers=2, max_seq=16, forward_mode=mode)
    eng = llama.LlamaEngine(cfg, init="device", comm=llama.NoPeers())
    forced = np.random.Generator(np.random.PCG64(1)).integers(0, cfg.vocab, 8)
    eng.reset(forced=forced)
    before = [bits(t.data) for t in eng.targets]
    eng.decode_step()
    dec = eng.decision()
    cur = (tuple(dec.expert_ids), tuple(dec.weights))
    print(mode, "chase", eng.chase, "split", eng.chase_split, "decision", cur)
    for i, t in enumerate(eng.targets):
        want = before[i].copy()
        orc.switch_segment_bf16(want, bits(eng.bank_down[i]), bits(eng.bank_up[i]), None, cur)
        got = bits(t.data)
        g, w = orc.from_bf16_bits(got).astype(np.float64), orc.from_bf16_bits(want).astype(np.float64)
        ulp = orc.bf16_ulp_of(np.maximum(np.abs(w), np.abs(orc.from_bf16_bits(before[i]))))
        bad = np.abs(g - w) > 2 * ulp
        rows, cols = np.nonzero(bad)
        msg = f"seg {i} {llama.SEGMENT_NAMES[i % 7]} {got.shape}: bad {bad.sum()}"
        if bad.any():
            msg += f" rows [{rows.min()},{rows.max()}] cols [{cols.min()},{cols.max()}] row%128 hist {np.bincount(rows % 128 // 32, minlength=4)} " \
                   f"col strips {np.unique(cols // 128)[:12]} row tiles {np.unique(rows // 128)[:12]}"
            # is the result explained by a subset of the experts?
            for sub in [(0, 1), (2, 3), (0,), (1,), (2,), (3,), (0, 1, 2), ()]:
                w2 = before[i].copy()
                if sub:
                    orc.switch_segment_bf16(w2, bits(eng.bank_down[i]), bits(eng.bank_up[i]), None,
                                            (tuple(cur[0][j] for j in sub), tuple(cur[1][j] for j in sub)))
                d2 = np.abs(g - orc.from_bf16_bits(w2).astype(np.float64)) > 2 * ulp
                msg += f"\n      experts {sub}: bad {int((d2 & bad).sum())} of the bad set, {int(d2.sum())} overall"
        print(msg, flush=True)
    del eng
