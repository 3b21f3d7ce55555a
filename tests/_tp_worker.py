"""Worker of test_gpu_llama.py::test_tp_two_processes_over_torch_distributed — launched by
`python -m torch.distributed.run --nproc-per-node TP`, one process per rank.  Every rank sits on cuda:0
(the test box has one GPU) and the process group is gloo, so the engine's real exchange layer
(`llama.Collectives` on torch.distributed: decision broadcast, int64/f32 all-reduces, argmax all-gather)
carries the calls between PROCESSES; on a multi-GPU box the same calls go over NCCL.  Mode "push": no all-reduce calls at
all inside the layers -- each rank's chained launches add their partial sums into the other PROCESS's accumulators through a
CUDA IPC mapping (`llama.PeerBuffer.ipc`) and wait on cross-process phase counters; the two contexts time-slice one GPU."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_11873_b200 import llama  # noqa: E402


def main():
    out_dir, forward_mode = sys.argv[1], sys.argv[2]
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    forced = np.random.Generator(np.random.PCG64(31)).integers(0, 512, 8)
    push = forward_mode == "push"      # the chase schedule with the all-reduce pushed from the epilogues over CUDA IPC mappings
    cfg = llama.preset("tiny", tp_size=world, tp_rank=rank, forward_mode="chase" if push else forward_mode, max_seq=16, n_heads=4,
                       n_kv_heads=4, tp_push=True if push else False)
    dev = torch.device("cuda", 0)
    eng = llama.LlamaEngine(cfg, init="host", peers=(lambda n: llama.PeerBuffer.ipc(n, dev)) if push else None)
    assert getattr(eng, "tp_push", False) == push and bool(getattr(eng, "chase_chained", False)) == push
    eng.reset(forced=forced)
    tokens, logits = [], []
    for _ in range(len(forced)):
        tokens.append(int(eng.decode_step()))
        logits.append(eng.logits.float().cpu().numpy().copy())
    if push:   # no library collective inside the step: the exchanges are the engine's own, and the step replays as a graph
        assert type(eng.step_comm) is llama.PeerCollectives and eng.graph_ok() and "steady" in eng._graphs
        assert int(eng.peer_comm.epochs[0].item()) == len(forced) and int(eng.peer_comm.epochs[2].item()) == len(forced)
    eng.finalize()
    dev = float(eng.max_backbone_deviation())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), tokens=np.asarray(tokens), logits=np.stack(logits), deviation=dev)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
