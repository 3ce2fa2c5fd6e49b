"""GPU parity: the n-gram drafter kernel vs vLLM golden outputs and the oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden

from oracle import ngram_oracle

pytestmark = pytest.mark.gpu


def run_kernel(contexts, min_n, max_n, k, stride=None):
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    B = len(contexts)
    stride = stride or max([len(c) for c in contexts] + [1])
    buf = np.zeros((B, stride), dtype=np.int32)
    for i, c in enumerate(contexts):
        buf[i, : len(c)] = c
    tok = torch.from_numpy(buf).cuda()
    lens = torch.tensor([len(c) for c in contexts], dtype=torch.int32, device="cuda")
    draft = torch.empty((B, k), dtype=torch.int32, device="cuda")
    nd = torch.empty(B, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(2 * B, dtype=torch.int64, device="cuda")
    for _ in range(2):  # second call checks the scratch was left zeroed
        _native.check(lib.sr_ngram_propose(B, tok.data_ptr(), stride, lens.data_ptr(), min_n,
                                           max_n, k, draft.data_ptr(), nd.data_ptr(),
                                           scratch.data_ptr(), _native.stream_handle()),
                      "sr_ngram_propose")
    torch.cuda.synchronize()
    assert int(scratch.abs().sum()) == 0
    d, n = draft.cpu().numpy(), nd.cpu().numpy()
    return [d[i, : n[i]].tolist() for i in range(B)]


def test_ngram_matches_vllm_golden():
    for case in golden("ngram_vllm.json"):
        if case["max_model_len"] != 100000:
            stride = case["max_model_len"]
        else:
            stride = max(len(case["ctx"]) + 16, 1)
        if stride < len(case["ctx"]) or stride < 1:
            continue
        got = run_kernel([case["ctx"]], case["min_n"], case["max_n"], case["k"], stride)[0]
        assert got == case["draft"], case


@pytest.mark.parametrize("length", [2, 100, 4097, 20000])
def test_ngram_batch_vs_oracle(length):
    rng = np.random.default_rng(length)
    ctxs = [rng.integers(0, int(rng.choice([3, 50, 5000])), size=int(rng.integers(1, length + 1)))
            for _ in range(16)]
    got = run_kernel(ctxs, 1, 3, 4, stride=length + 64)
    for c, g in zip(ctxs, got):
        assert g == ngram_oracle.propose(c, 1, 3, 4, length + 64)


def run_pooled(contexts, min_n, max_n, k, stride=None):
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    B = len(contexts)
    stride = stride or max([len(c) for c in contexts] + [1])
    buf = np.zeros((B, stride), dtype=np.int32)
    for i, c in enumerate(contexts):
        buf[i, : len(c)] = c
    tok = torch.from_numpy(buf).cuda()
    lens = torch.tensor([len(c) for c in contexts], dtype=torch.int32, device="cuda")
    draft = torch.empty((B, k), dtype=torch.int32, device="cuda")
    nd = torch.empty(B, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(2 * B, dtype=torch.int64, device="cuda")
    for _ in range(2):  # second call checks the scratch was left zeroed
        _native.check(lib.sr_pooled_ngram_propose(B, tok.data_ptr(), stride, lens.data_ptr(), min_n, max_n, k,
                                                  draft.data_ptr(), nd.data_ptr(), scratch.data_ptr(),
                                                  _native.stream_handle()), "sr_pooled_ngram_propose")
    torch.cuda.synchronize()
    assert int(scratch.abs().sum()) == 0
    d, n = draft.cpu().numpy(), nd.cpu().numpy()
    return [d[i, : n[i]].tolist() for i in range(B)]


@pytest.mark.parametrize("min_n,max_n,k", [(1, 3, 4), (2, 2, 3), (3, 4, 5), (1, 1, 2)])
def test_pooled_ngram_matches_oracle(min_n, max_n, k):
    """Grouped samples share spans: the pooled kernel equals the oracle's rule
    (own context first, then other rows in index order, earliest match)."""
    rng = np.random.default_rng(min_n * 10 + max_n)
    base = rng.integers(0, 5, 40)
    ctxs = []
    for i in range(12):
        n = int(rng.integers(1, 90))
        c = rng.integers(0, 5, n)
        if i % 3 == 0 and n > 20:        # a group sibling: shares a span of the base text
            o = int(rng.integers(0, n - 15))
            c[o:o + 15] = base[:15]
        ctxs.append(c.astype(np.int32))
    got = run_pooled(ctxs, min_n, max_n, k)
    for b in range(len(ctxs)):
        assert got[b] == ngram_oracle.propose_pooled(ctxs, b, min_n, max_n, k, max_model_len=max(map(len, ctxs))), b


def test_pooled_ngram_single_request_equals_ngram_kernel():
    rng = np.random.default_rng(5)
    for _ in range(20):
        c = rng.integers(0, 6, int(rng.integers(1, 200))).astype(np.int32)
        assert run_pooled([c], 1, 3, 4) == run_kernel([c], 1, 3, 4)


def test_pooled_drafter_in_engine_equals_plain():
    """Best-of-N with an n-gram and a pooled drafter over a group of prompts
    sharing text: committed tokens == plain greedy."""
    from paper_2511_16193_b200.engine import NgramDrafter, PooledNgramDrafter, RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    s = shape("tiny")
    rng = np.random.default_rng(11)
    shared = rng.integers(0, s.vocab, 24)
    prompts = [np.concatenate([rng.integers(0, s.vocab, 8), shared, rng.integers(0, s.vocab, 4)]).astype(np.int32)
               for _ in range(4)]
    max_new = [20, 14, 25, 9]
    B, K = len(prompts), 4
    m = DeviceModel(s, init_weights(s, seed=0), dtype="bf16", max_requests=B, max_len=128,
                    max_tokens=B * 2 * (K + 1), max_seqs=B * 2, branches=B)
    plain = RolloutEngine(m, prompts, max_new, k=0, history=1)
    plain.prefill()
    plain.run()
    eng = RolloutEngine(m, prompts, max_new, k=K, drafters=(NgramDrafter(), PooledNgramDrafter(1, 3)), history=1)
    eng.prefill()
    eng.run()
    assert eng.outputs() == plain.outputs()
