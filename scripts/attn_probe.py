"""Time K2 (paged verify attention) alone on controlled shapes.

    python scripts/attn_probe.py --ctx 128 512 1024 2048 --seqs 256
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_16193_b200 import _native  # noqa: E402


def run(lib, S, ctx, q_len, nq, nkv, hd, iters=20):
    pages_per = (ctx + q_len + 63) // 64 + 1
    P = S * pages_per
    cache = torch.randn(1, P, 2, nkv, 64, hd, device="cuda").bfloat16()
    btab = torch.arange(P, dtype=torch.int32, device="cuda").view(S, pages_per)
    M = S * q_len
    q = torch.randn(M, nq, hd, device="cuda").bfloat16()
    out = torch.empty_like(q)
    seqs = np.zeros((S, 8), np.int32)
    for s in range(S):
        seqs[s, :5] = (s * q_len, q_len, s, ctx, -1)
    seqs = torch.from_numpy(seqs).cuda()
    part = torch.empty(256 << 20, dtype=torch.float32, device="cuda")
    st = _native.stream_handle()
    max_key = ctx + q_len - 1

    def go():
        _native.check(lib.sr_paged_attention(1, q.data_ptr(), seqs.data_ptr(), S, q_len, max_key, nq, nkv, hd, 0, 1,
                                              cache.data_ptr(), P, btab.data_ptr(), pages_per, None, 0, 8,
                                              part.data_ptr(), part.numel(), out.data_ptr(), st), "attn")
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        go()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    kv_bytes = S * nkv * (ctx + q_len) * hd * 2 * 2
    return us, kv_bytes / us / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, nargs="+", default=[128, 512, 1024, 2048, 4096])
    ap.add_argument("--seqs", type=int, nargs="+", default=[256])
    ap.add_argument("--q", type=int, default=5)
    ap.add_argument("--heads", type=int, nargs=3, default=[12, 2, 128])
    ap.add_argument("--split", type=int, nargs="+", default=[16])
    a = ap.parse_args()
    lib = _native.lib()
    nq, nkv, hd = a.heads
    for sp in a.split:
        lib.sr_set_attention_split(sp)
        for S in a.seqs:
            for ctx in a.ctx:
                us, gbs = run(lib, S, ctx, a.q, nq, nkv, hd)
                print(f"split={sp:3d} S={S:4d} ctx={ctx:5d} q={a.q}: {us:8.1f} us  {gbs:7.0f} GB/s")


if __name__ == "__main__":
    main()
