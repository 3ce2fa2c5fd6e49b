"""Keyed deterministic random streams (host side).

Contract of ``pkg/src/specrollout/streams.py:16-30``: a stream is named by
``(seed, *keys)``; string keys hash to their CRC-32, integer keys are masked to
32 bits, and the words seed a numpy ``SeedSequence`` feeding PCG64.  The host
uses numpy for trace synthesis (``gen_trace``).  The per-position draws on the
rollout hot path (target tokens, acceptance uniforms) are regenerated on the
GPU by ``sr_keyed_tokens`` / ``sr_keyed_uniforms`` from the same words, see
``csrc/keyed_stream.cuh``; :func:`key_words` is the shared word encoding.
"""

from __future__ import annotations

import zlib

import numpy as np

MASK32 = 0xFFFFFFFF
MASK64 = 0xFFFFFFFFFFFFFFFF


def key_word(key: int | str) -> int:
    """One stream-name component as a 32-bit word."""
    if isinstance(key, str):
        return zlib.crc32(key.encode("utf-8"))
    return int(key) & MASK32


def key_words(seed: int, *keys: int | str) -> list[int]:
    """The SeedSequence entropy list of stream ``(seed, *keys)``."""
    return [int(seed) & MASK64] + [key_word(k) for k in keys]


def stream(seed: int, *keys: int | str) -> np.random.Generator:
    """Generator of the named ``(seed, *keys)`` stream."""
    return np.random.default_rng(np.random.SeedSequence(key_words(seed, *keys)))


def uniforms(seed: int, n: int, *keys: int | str) -> np.ndarray:
    """``n`` uniform [0, 1) doubles of the named stream."""
    return stream(seed, *keys).random(n)
