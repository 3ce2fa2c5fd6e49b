"""Pooled prompt lookup, oracle side: with one request the pooled rule is the
(vLLM-pinned) n-gram rule; hand-worked cross-request cases pin the tie order
(own context, then other requests in index order, then earliest match)."""

from __future__ import annotations

import numpy as np

from oracle import ngram_oracle


def test_single_request_equals_ngram_rule():
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 60))
        ctx = rng.integers(0, 6, n)
        for (lo, hi, k) in ((1, 3, 4), (2, 2, 3), (3, 4, 5), (1, 1, 2)):
            assert ngram_oracle.propose_pooled([ctx], 0, lo, hi, k) == ngram_oracle.propose(ctx, lo, hi, k)


def test_cross_request_match_and_tie_order():
    own = [9, 8, 1, 2, 3]                 # suffix ... 1 2 3, no earlier match in its own context
    other0 = [5, 1, 2, 3, 7, 7]           # match of length 3 ending at 3 -> continuation [7, 7]
    other2 = [1, 2, 3, 4, 4, 4]           # also length 3, later row -> loses the tie
    rows = [other0, own, other2]
    assert ngram_oracle.propose_pooled(rows, 1, 1, 3, 4) == [7, 7]
    # a longer match wins over row order
    rows = [other0, [6, 1, 2, 3], [6, 1, 2, 3, 9, 9]]
    assert ngram_oracle.propose_pooled(rows, 1, 1, 4, 2) == [9, 9]
    # the own context wins a tie
    own = [1, 2, 3, 5, 1, 2, 3]
    assert ngram_oracle.propose_pooled([other0, own], 1, 1, 3, 2) == [5, 1]
    # below min_n: nothing
    assert ngram_oracle.propose_pooled([[4, 4, 4], [1, 2, 3]], 1, 2, 3, 2) == []
