"""Verify-attention kernel in isolation at the bench workload's shape
(Qwen2.5-1.5B: 12 q heads, 2 kv heads, head_dim 128; 256 sequences, 5-row
verify windows, contexts U[128, 1024]): time per call and K/V bytes / time.
Two cache layers alternate so consecutive calls do not hit L2 (2 x 160 MB).

    python scripts/micro/attn_probe.py [--iters 50]

Measurement builds: SR_EXTRA_NVCC_FLAGS=-DSR_ATTN_PROBE=1 (loads only) / =2
(math only) rebuild the library with half of the kernel disabled.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

from paper_2511_16193_b200 import _native  # noqa: E402

PAGE = 64


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqs", type=int, default=256)
    ap.add_argument("--q-len", type=int, default=5)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--nq", type=int, default=12)
    ap.add_argument("--nkv", type=int, default=2)
    ap.add_argument("--hd", type=int, default=128)
    ap.add_argument("--ctx", type=int, nargs=2, default=[128, 1024], help="context range (inclusive)")
    a = ap.parse_args()
    lib = _native.lib()
    rng = np.random.default_rng(0)
    S, ql, nq, nkv, hd = a.seqs, a.q_len, a.nq, a.nkv, a.hd
    ctx = rng.integers(a.ctx[0], a.ctx[1] + 1, S)
    total = ctx + ql
    pages_per = (total + PAGE - 1) // PAGE
    P = int(pages_per.sum())
    max_pages = int(pages_per.max())
    btab = np.zeros((S, max_pages), np.int32)
    nxt = 0
    for s in range(S):
        btab[s, :pages_per[s]] = np.arange(nxt, nxt + pages_per[s])
        nxt += pages_per[s]
    dev = "cuda"
    layers = 2
    cache = (torch.randn(layers, P, 2, nkv, PAGE * hd, device=dev) * 0.5).to(torch.bfloat16)
    window = torch.zeros(layers, 1, 2, nkv, 8 * hd, dtype=torch.bfloat16, device=dev)
    seqs = np.zeros((S, 8), np.int32)
    for s in range(S):
        seqs[s, :5] = (s * ql, ql, s, ctx[s], -1)
    seqs_d = torch.from_numpy(seqs).to(dev)
    btab_d = torch.from_numpy(btab).to(dev)
    q = torch.randn(S * ql, nq, hd, device=dev).to(torch.bfloat16)
    out = torch.zeros_like(q)
    part = torch.zeros(64 << 20, dtype=torch.float32, device=dev)
    max_key = int((ctx + ql - 1).max())
    stream = _native.stream_handle()

    def call(layer):
        _native.check(lib.sr_paged_attention(
            1, q.data_ptr(), seqs_d.data_ptr(), S, ql, max_key, nq, nkv, hd, layer, layers, cache.data_ptr(), P,
            btab_d.data_ptr(), max_pages, window.data_ptr(), 1, 8, part.data_ptr(), part.numel(), out.data_ptr(),
            stream), "attention")

    for i in range(5):
        call(i % 2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ = torch.cuda.current_stream()
    e0.record(s_)
    for i in range(a.iters):
        call(i % 2)
    e1.record(s_)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.iters
    tiles = int(((ctx + ql - 1) // PAGE + 1).sum()) * nkv
    kv_bytes = tiles * PAGE * hd * 2 * 2
    print(json.dumps({"us_per_call": round(us, 2), "kv_mb": round(kv_bytes / 1e6, 1),
                      "gb_per_s": round(kv_bytes / us / 1e3, 1), "tiles": tiles,
                      "finite": bool(torch.isfinite(out.float()).all())}))


if __name__ == "__main__":
    main()
