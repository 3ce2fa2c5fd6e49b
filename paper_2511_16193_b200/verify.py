"""Device state of a reference-semantics ("truth" mode) rollout.

The reference derives every target token and acceptance draw from keyed
numpy streams (``sim.py:313-336``).  :class:`DeviceVerifier` materializes
those streams once, on the GPU, as a truth table ``[R, L]`` and a uniform
table ``[R, M, L]`` (``sr_keyed_tokens`` / ``sr_keyed_uniforms``), then
serves each executor round with one ``sr_verify_windows`` launch that
updates the device token buffer ``seq`` and the committed-high watermark.
Host traffic per round is the window descriptors in and four int32 per
window out.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native
from .streams import MASK32, key_word

VOCAB = 50_257
CHUNK = 256


def entropy_words(seed: int, *keys) -> list[int]:
    """numpy ``SeedSequence`` coercion of ``[seed, *keys]`` to uint32 words."""
    s = int(seed) & 0xFFFFFFFFFFFFFFFF
    words = [0] if s == 0 else []
    while s > 0:
        words.append(s & MASK32)
        s >>= 32
    return words + [key_word(k) for k in keys]


def _word_table(rows: list[list[int]]):
    width = max(len(r) for r in rows)
    table = np.zeros((len(rows), width), dtype=np.uint32)
    counts = np.array([len(r) for r in rows], dtype=np.int32)
    for i, r in enumerate(rows):
        table[i, : len(r)] = r
    return table, counts, width


def keyed_fill(kind: str, streams: list[list[int]], per_stream: int,
               out: torch.Tensor, high: int = VOCAB) -> None:
    """Fill ``out`` (device, ``[S, per_stream]``) with the named streams."""
    lib = _native.lib()
    if not streams:
        return
    table, counts, width = _word_table(streams)
    dev = out.device
    words = torch.from_numpy(table.view(np.int32)).to(dev)
    nw = torch.from_numpy(counts).to(dev)
    st = _native.stream_handle()
    if kind == "tokens":
        _native.check(lib.sr_keyed_tokens(len(streams), words.data_ptr(), nw.data_ptr(),
                                          width, high, per_stream, out.data_ptr(), st),
                      "sr_keyed_tokens")
    else:
        _native.check(lib.sr_keyed_uniforms(len(streams), words.data_ptr(), nw.data_ptr(),
                                            width, per_stream, out.data_ptr(), st),
                      "sr_keyed_uniforms")


def truth_table(seed: int, request_ids: list[int], lengths: list[int],
                device="cuda") -> torch.Tensor:
    """Target tokens ``[R, stride]`` of ``generate_true_sequence`` on device."""
    chunks = max([math.ceil(L / CHUNK) for L in lengths] + [1])
    out = torch.empty((len(request_ids), chunks * CHUNK), dtype=torch.int32, device=device)
    streams = [entropy_words(seed, rid, "tokens", c)
               for rid in request_ids for c in range(chunks)]
    keyed_fill("tokens", streams, CHUNK, out)
    return out


def keyed_true_tokens(seed: int, request_ids: list[int], lengths: list[int]) -> list[list[int]]:
    table = truth_table(seed, request_ids, lengths).cpu().numpy()
    return [table[i, :L].tolist() for i, L in enumerate(lengths)]


class DeviceVerifier:
    """Truth/uniform tables + token buffer for one rollout, on ``cuda``."""

    def __init__(self, seed: int, requests, methods: list[str], bonus_token: bool,
                 device: str = "cuda"):
        _native.lib()
        self.lib = _native.load()
        self.dev = torch.device(device)
        R, M = len(requests), len(methods)
        self.R, self.M = R, M
        lengths = [r.true_len for r in requests]
        chunks = max([math.ceil(L / CHUNK) for L in lengths] + [1])
        self.stride = chunks * CHUNK
        self.bonus = 1 if bonus_token else 0
        ids = [r.id for r in requests]
        self.truth = truth_table(seed, ids, lengths, self.dev)
        self.uniforms = torch.empty((R, M, self.stride), dtype=torch.float64, device=self.dev)
        if R:
            streams = [entropy_words(seed, rid, "accept_draw", m, c)
                       for rid in ids for m in methods for c in range(chunks)]
            keyed_fill("uniforms", streams, CHUNK, self.uniforms)
        p = np.full((R, M), np.nan, dtype=np.float64)
        for i, r in enumerate(requests):
            for j, m in enumerate(methods):
                if m in r.latent_accept:
                    p[i, j] = r.latent_accept[m]
        self.accept_p = torch.from_numpy(p).to(self.dev)
        self.true_len = torch.tensor(lengths, dtype=torch.int32, device=self.dev)
        self.seq = torch.full((R, self.stride), -1, dtype=torch.int32, device=self.dev)
        self.high = torch.zeros(R, dtype=torch.int32, device=self.dev)
        cap = max(R, 1)
        # flat buffers so a [4, W] prefix view is contiguous for any W
        self._win_h = torch.empty(4 * cap, dtype=torch.int32).pin_memory()
        self._out_h = torch.empty(4 * cap, dtype=torch.int32).pin_memory()
        self._win_d = torch.empty(4 * cap, dtype=torch.int32, device=self.dev)
        self._out_d = torch.empty(4 * cap, dtype=torch.int32, device=self.dev)

    def verify(self, rows, method: int, starts, ns, extra_waste):
        W = len(rows)
        win_h = self._win_h[: 4 * W].view(4, W)
        win = win_h.numpy()
        win[0], win[1], win[2], win[3] = rows, starts, ns, extra_waste
        win_d = self._win_d[: 4 * W].view(4, W)
        win_d.copy_(win_h, non_blocking=True)
        out_d = self._out_d[: 4 * W].view(4, W)
        st = _native.stream_handle()
        _native.check(self.lib.sr_verify_windows(
            W, win_d.data_ptr(), method, self.M, self.stride, self.truth.data_ptr(),
            self.uniforms.data_ptr(), self.accept_p.data_ptr(), self.true_len.data_ptr(),
            self.bonus, self.seq.data_ptr(), self.high.data_ptr(), out_d.data_ptr(), st),
            "sr_verify_windows")
        host = self._out_h[: 4 * W].view(4, W)
        host.copy_(out_d, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        res = host.numpy().copy()
        return res[0], res[1], res[2], res[3]

    def sequences(self) -> list[list[int]]:
        return self.seq.cpu().numpy().tolist()
