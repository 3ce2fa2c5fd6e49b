"""CPU ORACLE (test infrastructure only) for the n-gram drafter.

Restates vLLM 0.22's ``_find_longest_matched_ngram_and_propose_tokens``
(vllm/v1/spec_decode/ngram_proposer.py:198-285; the paper's n-gram drafter,
PAPER.md:1668-1681) as a direct brute force: for each candidate start s
(match ending at or before len-2) the longest n <= max_n with
ctx[s:s+n] == ctx[len-n:len]; keep the longest, earliest s on ties; propose
up to min(k, max_model_len - len, tokens after the match).  Pinned against
vLLM's own outputs in tests/golden/ngram_vllm.json.
"""

from __future__ import annotations

import numpy as np


def propose(ctx, min_n: int, max_n: int, k: int, max_model_len: int | None = None) -> list[int]:
    ctx = np.asarray(ctx)
    total = len(ctx)
    if max_model_len is None:
        max_model_len = 1 << 40
    if total < min_n:
        return []
    k = min(k, max_model_len - total)
    if k <= 0:
        return []
    best_n, best_s = 0, -1
    for s in range(total - 1):
        n = 0
        # match ctx[s .. s+n) against the suffix of length n; the match must
        # end at or before position total-2
        for cand in range(1, max_n + 1):
            if s + cand - 1 > total - 2:
                break
            if np.array_equal(ctx[s:s + cand], ctx[total - cand:]):
                n = cand
        if n > best_n:
            best_n, best_s = n, s
    if best_n < min_n:
        return []
    start = best_s + best_n
    k = min(k, total - start)
    return [int(x) for x in ctx[start:start + k]]


def propose_pooled(rows, b: int, min_n: int, max_n: int, k: int, max_model_len: int | None = None) -> list[int]:
    """Pooled prompt lookup (``sr_pooled_ngram_propose``): request ``b``'s
    suffix against its own context (exactly :func:`propose`'s rule) and every
    other request's tokens ``rows[r]``.  Longest match length n in [min_n,
    max_n] wins; ties: own context, then other rows in index order, then the
    earliest match.  Up to k tokens following the match in its row.  Test
    infrastructure only."""
    own = np.asarray(rows[b])
    total = len(own)
    if max_model_len is None:
        max_model_len = 1 << 40
    if total < min_n:
        return []
    k = min(k, max_model_len - total)
    if k <= 0:
        return []
    order = [b] + [r for r in range(len(rows)) if r != b]
    best = (0, None, -1)   # (n, row, start)
    for r in order:
        ctx = np.asarray(rows[r])
        end_lim = (total if r == b else len(ctx)) - 2   # a continuation token must follow
        for s in range(len(ctx)):
            n = 0
            for cand in range(1, max_n + 1):
                if s + cand - 1 > end_lim or cand > total:
                    break
                if np.array_equal(ctx[s:s + cand], own[total - cand:]):
                    n = cand
            if n > best[0]:
                best = (n, r, s)
    n, r, s = best
    if n < min_n or r is None:
        return []
    ctx = np.asarray(rows[r])
    start = s + n
    k = min(k, len(ctx) - start)
    return [int(x) for x in ctx[start:start + k]]
