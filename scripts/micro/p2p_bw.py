"""NCCL point-to-point bandwidth between two ranks (the transport under
request migration and decoupled mode): one send/recv of S bytes, timed with
CUDA events on the sender, after warm-up.

    torchrun --nproc-per-node 2 scripts/micro/p2p_bw.py
"""

import json
import os

import torch
import torch.distributed as dist


def main():
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    peer = 1 - rank
    for mb in (1, 16, 64, 256):
        x = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
        for _ in range(3):
            (dist.send if rank == 0 else dist.recv)(x, peer)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            (dist.send if rank == 0 else dist.recv)(x, peer)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        if rank == 0:
            print(json.dumps({"MB": mb, "ms": round(ms, 4), "GB_per_s": round((mb << 20) / ms / 1e6, 1)}))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
