"""GPU parity of K2 (paged GQA verify attention) on its own: ragged contexts
up to 5 KV splits (combine kernel), non-contiguous block tables, partial last
pages, drafter-branch window keys, head_dim 64 and 128, bf16 and fp32 caches
-- against a float64 torch reference of causal softmax attention -- plus the
batch-invariance property the exactness invariant rests on (a query's output
is bit-identical whether it is verified in a 5-position window or decoded
alone)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

PAGE = 64


def kv_index(slot, d, rows, hd, bf16):
    """Element offset of (slot, d) in one [rows, hd] head block (layers.cuh kv_off)."""
    if not bf16:
        return slot * hd + d
    return ((d >> 3) ^ (slot & 7)) * 8 + (d & 7) + slot * hd


def build_case(seed, S, ctx, q_len, nq, nkv, hd, dtype, branches=None):
    """Random sequences + their K/V written into a shuffled paged cache (and
    branch windows for sequences with a branch)."""
    g = torch.Generator().manual_seed(seed)
    bf16 = dtype == torch.bfloat16
    total = [c + q for c, q in zip(ctx, q_len)]
    pages_per = [(t + PAGE - 1) // PAGE for t in total]
    P = sum(pages_per) + 3
    perm = torch.randperm(P, generator=g).tolist()
    max_pages = max(pages_per)
    btab = torch.zeros((S, max_pages), dtype=torch.int32)
    cache = torch.zeros((1, P, 2, nkv, PAGE * hd), dtype=dtype)
    wmax = max(q_len) + 1
    nbr = max(1, len([b for b in (branches or []) if b >= 0]))
    window = torch.zeros((1, nbr, 2, nkv, wmax * hd), dtype=dtype)
    K, V, Q = [], [], []
    nxt = 0
    for s in range(S):
        k = torch.randn(total[s], nkv, hd, generator=g)
        v = torch.randn(total[s], nkv, hd, generator=g)
        K.append(k), V.append(v)
        Q.append(torch.randn(q_len[s], nq, hd, generator=g))
        for pg in range(pages_per[s]):
            btab[s, pg] = perm[nxt]
            nxt += 1
        br = branches[s] if branches else -1
        idx = torch.tensor([kv_index(sl, d, PAGE, hd, bf16) for sl in range(PAGE) for d in range(hd)])
        widx = torch.tensor([kv_index(sl, d, wmax, hd, bf16) for sl in range(wmax) for d in range(hd)])
        for pos in range(total[s]):
            if br >= 0 and pos >= ctx[s]:
                j = pos - ctx[s]
                for sel, t in ((0, k), (1, v)):
                    window[0, br, sel, :, widx.view(wmax, hd)[j]] = t[pos].to(dtype)
            else:
                page, slot = int(btab[s, pos // PAGE]), pos % PAGE
                for sel, t in ((0, k), (1, v)):
                    cache[0, page, sel, :, idx.view(PAGE, hd)[slot]] = t[pos].to(dtype)
    return dict(K=K, V=V, Q=Q, cache=cache, btab=btab, window=window, wmax=wmax, nbr=nbr, P=P,
                max_pages=max_pages)


def reference(case, ctx, q_len, nq, nkv, hd, dtype):
    G = nq // nkv
    outs = []
    for s, q in enumerate(case["Q"]):
        k = case["K"][s].to(dtype).double()
        v = case["V"][s].to(dtype).double()
        qq = q.to(dtype).double()
        o = torch.zeros_like(qq)
        for j in range(q_len[s]):
            n = ctx[s] + j + 1
            for h in range(nq):
                sc = k[:n, h // G] @ qq[j, h] / np.sqrt(hd)
                p = torch.softmax(sc, 0)
                o[j, h] = p @ v[:n, h // G]
        outs.append(o)
    return torch.cat(outs)


@pytest.fixture(params=["mma_sync", "tcgen05"], autouse=True)
def attention_kernel(request):
    """Every case runs on both head_dim-128 kernels (mma.sync default and
    the tcgen05/TMEM kernel); SR_ATTN_TC_GRID (set by the harness) caps the
    tcgen05 grid so CTAs chain several items."""
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    _native.check(lib.sr_set_attention_tc(1 if request.param == "tcgen05" else 0), "kernel")
    yield request.param
    _native.check(lib.sr_set_attention_tc(0), "kernel")


def run_gpu(case, ctx, q_len, nq, nkv, hd, dtype, branches=None, split=32):
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    S = len(ctx)
    seqs = np.zeros((S, 8), np.int32)
    start = 0
    for s in range(S):
        seqs[s, :5] = (start, q_len[s], s, ctx[s], branches[s] if branches else -1)
        start += q_len[s]
    dev = "cuda"
    q = torch.cat(case["Q"]).to(dtype).to(dev).contiguous()
    out = torch.zeros_like(q)
    cache = case["cache"].to(dev)
    window = case["window"].to(dev)
    btab = case["btab"].to(dev)
    seqs_d = torch.from_numpy(seqs).to(dev)
    part = torch.zeros(32 << 20, dtype=torch.float32, device=dev)
    max_key = max(c + l - 1 for c, l in zip(ctx, q_len))
    _native.check(lib.sr_set_attention_split(split), "split")
    _native.check(lib.sr_paged_attention(
        1 if dtype == torch.bfloat16 else 0, q.data_ptr(), seqs_d.data_ptr(), S, max(q_len), max_key, nq, nkv, hd,
        0, 1, cache.data_ptr(), case["P"], btab.data_ptr(), case["max_pages"], window.data_ptr(), case["nbr"],
        case["wmax"], part.data_ptr(), part.numel(), out.data_ptr(), _native.stream_handle()), "attention")
    torch.cuda.synchronize()
    _native.check(lib.sr_set_attention_split(32), "split")
    return out.cpu()


CASES = [
    # (ctx per sequence, q_len per sequence, nq, nkv, hd)
    ([0, 5, 63, 64, 65, 200], [1, 2, 5, 5, 3, 4], 12, 2, 128),     # page edges, short
    ([2040, 2047, 2048, 4100, 9000], [5, 1, 5, 3, 2], 12, 2, 128),  # 1..5 KV splits -> combine
    ([130, 777, 3000], [5, 5, 5], 14, 2, 64),                        # head_dim 64, G = 7
    ([0, 0, 300], [100, 1, 64], 12, 2, 128),                          # prefill: 32-row blocks across tokens
    ([500, 1500, 2100], [5, 5, 5], 28, 4, 128),                       # 7B shape: G = 7, two row blocks
    ([64, 1000, 4095], [5, 5, 5], 40, 8, 128),                        # 32B shape: G = 5
    ([20000, 16385], [5, 1], 12, 2, 128),                             # 20K-key long tail: 10 splits
]


@pytest.mark.parametrize("ctx,q_len,nq,nkv,hd", CASES)
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_attention_vs_float64_reference(ctx, q_len, nq, nkv, hd, dtype):
    if dtype == torch.float32 and max(ctx) > 5000:
        pytest.skip("fp32 parity path: per-(token, head) warp loop, keep it short")
    case = build_case(1, len(ctx), ctx, q_len, nq, nkv, hd, dtype)
    got = run_gpu(case, ctx, q_len, nq, nkv, hd, dtype).double()
    exp = reference(case, ctx, q_len, nq, nkv, hd, dtype)
    tol = 1e-2 if dtype == torch.bfloat16 else 1e-5
    torch.testing.assert_close(got, exp, rtol=tol, atol=tol)


def test_attention_branch_window_keys():
    """Best-of-N drafter branches: keys >= ctx_len come from the branch window."""
    ctx, q_len, nq, nkv, hd = [100, 2100, 64], [5, 4, 5], 12, 2, 128
    branches = [0, -1, 1]
    case = build_case(2, 3, ctx, q_len, nq, nkv, hd, torch.bfloat16, branches=branches)
    got = run_gpu(case, ctx, q_len, nq, nkv, hd, torch.bfloat16, branches=branches).double()
    exp = reference(case, ctx, q_len, nq, nkv, hd, torch.bfloat16)
    torch.testing.assert_close(got, exp, rtol=1e-2, atol=1e-2)


def test_attention_verify_window_equals_single_decode_bit_exact():
    """A query's output is the same bits in a 5-position verify window and
    as a 1-position decode step, including across the split boundary."""
    nq, nkv, hd = 12, 2, 128
    for ctx0 in (70, 2045):
        ctx, q_len = [ctx0], [5]
        case = build_case(3, 1, ctx, q_len, nq, nkv, hd, torch.bfloat16)
        full = run_gpu(case, ctx, q_len, nq, nkv, hd, torch.bfloat16)
        for j in range(5):
            one = dict(case, Q=[case["Q"][0][j:j + 1]])
            single = run_gpu(one, [ctx0 + j], [1], nq, nkv, hd, torch.bfloat16)
            assert torch.equal(single[0], full[j]), (ctx0, j)


@pytest.mark.parametrize("split", [4, 6, 5])
def test_attention_split_sizes(split):
    """Non-default split sizes: even sizes keep the tcgen05 kernel's 128-key
    blocks split aligned, odd sizes fall back to the mma.sync kernel."""
    ctx, q_len, nq, nkv, hd = [300, 900, 1700], [5, 3, 5], 12, 2, 128
    case = build_case(4, 3, ctx, q_len, nq, nkv, hd, torch.bfloat16)
    got = run_gpu(case, ctx, q_len, nq, nkv, hd, torch.bfloat16, split=split).double()
    exp = reference(case, ctx, q_len, nq, nkv, hd, torch.bfloat16)
    torch.testing.assert_close(got, exp, rtol=1e-2, atol=1e-2)


def test_attention_tcgen05_items_chained_per_cta(monkeypatch, attention_kernel):
    """Three CTAs for ~90 work items: every CTA chains many items through its
    pipelines (item ring, Q buffers, S/O slots, end-of-work sentinel)."""
    if attention_kernel != "tcgen05":
        pytest.skip("grid cap applies to the tcgen05 kernel")
    monkeypatch.setenv("SR_ATTN_TC_GRID", "3")
    ctx = [0, 5, 63, 64, 65, 200, 700, 1500, 2047, 2100, 3000, 90, 128, 129, 333]
    q_len = [1, 2, 5, 5, 3, 4, 5, 5, 1, 5, 2, 5, 5, 1, 4]
    nq, nkv, hd = 12, 2, 128
    case = build_case(5, len(ctx), ctx, q_len, nq, nkv, hd, torch.bfloat16)
    got = run_gpu(case, ctx, q_len, nq, nkv, hd, torch.bfloat16).double()
    exp = reference(case, ctx, q_len, nq, nkv, hd, torch.bfloat16)
    torch.testing.assert_close(got, exp, rtol=1e-2, atol=1e-2)
