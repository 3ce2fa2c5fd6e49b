"""Cross-GPU request migration over NCCL P2P (NVLink): rank 0 runs a rollout,
ships `--move` requests (tokens + lengths + KV pages) to rank 1 mid-flight,
rank 1 finishes them; outputs are checked against plain decoding and the
transfer is timed (replaces the reference's 50 ms + 0.01 ms/token scale-cost
model, scenarios.py:84-88).

    torchrun --nproc-per-node 2 scripts/migrate_ranks.py [--model qwen2.5-1.5b]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine  # noqa: E402
from paper_2511_16193_b200.migrate import recv_requests, send_requests  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--move", type=int, default=8)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    s = shape(a.model, a.layers)
    rng = np.random.default_rng(0)
    words = rng.integers(0, s.vocab, 64)
    prompts = [words[rng.integers(0, 64, int(rng.integers(600, 1000)))].astype(np.int32) for _ in range(a.batch)]
    max_new = [int(x) for x in rng.integers(40, 80, a.batch)]
    m = DeviceModel(s, init_weights(s, seed=0, device="cuda"), dtype="bf16", max_requests=a.batch,
                    max_len=1200, max_tokens=a.batch * 5, max_seqs=a.batch)
    eng = RolloutEngine(m, prompts, max_new, k=4, drafters=(NgramDrafter(),), history=1)
    eng.prefill()
    moved = list(range(a.move))
    res = {"rank": rank}
    warm = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")   # NCCL connection setup, both paths
    peer = 1 - rank
    if rank == 0:
        dist.send(warm, peer)
    else:
        dist.recv(warm, peer)
    op = dist.P2POp(dist.isend if rank == 0 else dist.irecv, warm, peer)
    for w in dist.batch_isend_irecv([op]):
        w.wait()
    pool = torch.empty(640 << 20, dtype=torch.uint8, device="cuda")   # warm the caching allocator
    del pool
    if rank == 0:
        for _ in range(a.steps):
            eng.step()
        torch.cuda.synchronize()
        dist.barrier()
        from paper_2511_16193_b200.migrate import pack_request
        sts = [pack_request(eng, b) for b in moved]      # untimed: first-use gather / allocator warm-up
        kv = torch.cat([st["kv"] for st in sts], 1)
        torch.cuda.synchronize()
        del sts, kv
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nbytes = send_requests(dist, eng, moved, 1)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res.update(bytes=nbytes, ms=ms, gb_per_s=nbytes / ms / 1e6,
                   tokens=int(sum(int(eng.seq_len[b]) for b in moved)))
    else:
        plain = RolloutEngine(m, prompts, max_new, k=0, drafters=(NgramDrafter(),), history=1)
        plain.prefill()
        plain.run()
        ref = plain.outputs()
        eng2 = RolloutEngine(m, prompts, max_new, k=4, drafters=(NgramDrafter(),), history=1)
        eng2.prefill()
        torch.cuda.synchronize()
        dist.barrier()
        recv_requests(dist, eng2, moved, 0)
        for b in range(a.move, a.batch):
            eng2.max_new[b] = eng2.gen_len[b]     # only the migrated requests continue here
        eng2.run()
        out = eng2.outputs()
        res["outputs_equal_plain"] = all(out[b] == ref[b] for b in moved)
    print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
