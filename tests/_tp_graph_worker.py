"""Worker of test_gpu_llama.py::test_tp_step_with_nccl_collectives_captures.  One process, a ONE-rank NCCL
group, a tp_size = 2 shard engine (rank 0) whose exchange layer is the shipped `llama.Collectives`: the
broadcast, all-reduces and all-gather go through torch's NCCL process group (identity on one rank — the
shard's numbers are not the model's, only the mechanics are under test).  The step is run eagerly, then
captured as a CUDA graph (AF_TP_GRAPH=1) and replayed: same tokens, same weights."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_11873_b200 import llama  # noqa: E402


def push_over_symmetric_memory(port):
    """`push` mode: the TP-push step with its accumulators in torch SYMMETRIC MEMORY (what maps the ranks' buffers into
    each other over NVLink), on a one-rank NCCL group: allocation, rendezvous and the peer offsets are the real ones,
    the only peer is the rank itself.  Bit-identical to the plain engine."""
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=dev)
    forced = np.random.Generator(np.random.PCG64(13)).integers(0, 512, 12)
    runs = []
    for push in (False, True):
        cfg = llama.preset("tiny", forward_mode="chase", max_seq=48, tp_push=push)
        eng = llama.LlamaEngine(cfg, init="host", peers=(lambda n: llama.PeerBuffer.symmetric(n, dev)) if push else None)
        assert eng.tp_push == push
        if push:
            assert eng.peer_buf.offsets == [0] and eng.peer_buf._keep is not None
        eng.reset(forced=forced)
        toks = [eng.decode_step() for _ in forced]
        runs.append((toks, [t.data.clone() for t in eng.targets]))
    assert runs[0][0] == runs[1][0], runs
    for ta, tb in zip(runs[0][1], runs[1][1]):
        assert torch.equal(ta, tb)
    dist.destroy_process_group()
    print("TP_PUSH_SYMM_OK")


def main():
    forward_mode, port = sys.argv[1], sys.argv[2]
    if forward_mode == "push":
        return push_over_symmetric_memory(port)
    os.environ["AF_TP_GRAPH"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    cfg = llama.preset("tiny", tp_size=2, tp_rank=0, forward_mode=forward_mode, max_seq=48, n_heads=4, n_kv_heads=4)
    forced = np.random.Generator(np.random.PCG64(12)).integers(0, cfg.vocab, 20)
    a = llama.LlamaEngine(cfg, init="host")
    assert a.comm.tp_size == 2 and type(a.comm) is llama.Collectives
    a.reset(forced=forced)
    for _ in range(20):
        a.decode_step()
    eager = a.tokens()
    b = llama.LlamaEngine(cfg, init="host")
    b.reset(forced=forced)
    b.decode_step()
    b.decode_step()
    b.capture()
    for _ in range(18):
        b.replay()
    torch.cuda.synchronize()
    assert b.tokens() == eager, (b.tokens(), eager)
    for ta, tb in zip(a.targets, b.targets):
        assert torch.equal(ta.data, tb.data)
    dist.destroy_process_group()
    print("TP_GRAPH_OK")


if __name__ == "__main__":
    main()
