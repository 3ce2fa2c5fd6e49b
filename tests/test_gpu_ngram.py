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
