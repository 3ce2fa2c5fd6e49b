"""CPU ORACLE (test infrastructure only) for keyed sampling.

Restates paper_2511_16193_b200/csrc/sampling.cuh in numpy: Philox4x32-10
keyed by (seed, request), counter (position, v // 4, 0x53414D50, 0); u = odd
multiple of 2^-24 from the top 23 bits; Gumbel G = -log(-log(u)) in float32;
token = argmax_v logit[v] / T + G[v] (lowest index on ties).  The reference
draws every target token from a position-keyed stream (sim.py:313-320); this
is the model-mode equivalent that keeps speculative == plain under T > 0.
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    c = [np.asarray(x, dtype=np.uint64) & MASK for x in (c0, c1, c2, c3)]
    k0, k1 = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for _ in range(10):
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ np.uint64(k0), lo1, hi0 ^ c[3] ^ np.uint64(k1), lo0]
        k0 = (k0 + W0) & 0xFFFFFFFF
        k1 = (k1 + W1) & 0xFFFFFFFF
    return [x.astype(np.uint32) for x in c]


def gumbel(seed: int, req: int, pos: int, vocab: int) -> np.ndarray:
    blocks = np.arange((vocab + 3) // 4, dtype=np.uint64)
    out = philox4x32_10(np.full_like(blocks, pos), blocks, np.full_like(blocks, 0x53414D50),
                        np.zeros_like(blocks), seed, req)
    x = np.stack(out, axis=1).reshape(-1)[:vocab]
    u = (((x >> np.uint32(9)) << np.uint32(1)) | np.uint32(1)).astype(np.float32) * np.float32(2.0 ** -24)
    return -np.log(-np.log(u))


def sample(logits_row, seed: int, req: int, pos: int, temperature: float) -> int:
    lg = np.asarray(logits_row, dtype=np.float32)
    v = lg * np.float32(1.0 / temperature) + gumbel(seed, req, pos, lg.shape[0])
    return int(np.argmax(v))
