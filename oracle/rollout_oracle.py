"""CPU ORACLE (test infrastructure only) for the verify/commit hot path.

Plain numpy restatement of the reference's per-window semantics:

* target token     -- ``sim.py:313-320``: stream(seed, rid, "tokens",
                      pos // 256).integers(0, 50257, 256)[pos % 256]
* acceptance draw  -- ``sim.py:322-336``: stream(seed, rid, "accept_draw",
                      method, pos // 256).random(256)[pos % 256] < p
* accepted prefix  -- ``sim.py:977-981``
* commit / waste   -- ``sim.py:983-1010`` (full accept: n [+ bonus]; partial:
                      a + 1, waste n - a - 1 + depth-2 successor)
* committed high   -- ``sim.py:340-353``
* plain step       -- ``sim.py:966-975`` (n == 0 here)

``OracleVerifier`` has the interface of the product's ``DeviceVerifier`` so
the host engine can be exercised on CPU and the kernel compared window by
window.  Streams use numpy directly: numpy 2.3.5's SeedSequence/PCG64 is the
reference's own dependency, so draws are the reference's bit for bit.
"""

from __future__ import annotations

import zlib

import numpy as np

VOCAB = 50_257
CHUNK = 256


def _stream(seed, *keys):
    words = [seed & 0xFFFFFFFFFFFFFFFF] + [
        zlib.crc32(k.encode()) if isinstance(k, str) else k & 0xFFFFFFFF for k in keys]
    return np.random.default_rng(np.random.SeedSequence(words))


def true_tokens(seed: int, rid: int, length: int) -> np.ndarray:
    chunks = -(-length // CHUNK)
    parts = [_stream(seed, rid, "tokens", c).integers(0, VOCAB, size=CHUNK)
             for c in range(chunks)]
    return np.concatenate(parts)[:length] if parts else np.zeros(0, np.int64)


def accept_uniforms(seed: int, rid: int, method: str, length: int) -> np.ndarray:
    chunks = -(-length // CHUNK)
    parts = [_stream(seed, rid, "accept_draw", method, c).random(CHUNK)
             for c in range(chunks)]
    return np.concatenate(parts)[:length] if parts else np.zeros(0)


def verify_window(u: np.ndarray, p: float, start: int, n: int, extra: int,
                  true_len: int, bonus: bool):
    """(accepted, committed, wasted) of one window."""
    if n == 0:
        return 0, 1, 0
    a = 0
    while a < n and u[start + a] < p:
        a += 1
    if a == n:
        return a, n + (1 if bonus and start + n < true_len else 0), 0
    return a, a + 1, max(n - a - 1, 0) + extra


class OracleVerifier:
    """CPU checker with the DeviceVerifier interface."""

    def __init__(self, seed, requests, methods, bonus_token, **_):
        self.bonus = bool(bonus_token)
        self.lens = [r.true_len for r in requests]
        self.truth = [true_tokens(seed, r.id, r.true_len) for r in requests]
        self.u = [[accept_uniforms(seed, r.id, m, r.true_len) for m in methods]
                  for r in requests]
        self.p = [[r.latent_accept.get(m, float("nan")) for m in methods] for r in requests]
        self.seq = [np.full(L, -1, dtype=np.int64) for L in self.lens]
        self.high = [0] * len(requests)

    def verify(self, rows, method, starts, ns, extra_waste):
        W = len(rows)
        out = np.zeros((4, W), dtype=np.int64)
        for i in range(W):
            r, start, n = int(rows[i]), int(starts[i]), int(ns[i])
            L = self.lens[r]
            a, c, w = verify_window(self.u[r][method], self.p[r][method], start, n,
                                    int(extra_waste[i]), L, self.bonus)
            conflict = False
            for j in range(c):
                pos = start + j
                tok = self.truth[r][pos]
                if self.seq[r][pos] < 0:
                    self.seq[r][pos] = tok
                elif self.seq[r][pos] != tok:
                    conflict = True
            h = self.high[r]
            while h < L and self.seq[r][h] >= 0:
                h += 1
            self.high[r] = h
            out[:, i] = (a, c, w, -1 if conflict else h)
        return out[0], out[1], out[2], out[3]

    def sequences(self):
        return [s.tolist() for s in self.seq]
