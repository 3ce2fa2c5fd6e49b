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
