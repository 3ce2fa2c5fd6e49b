"""GPU numerics: the tcgen05 bf16 GEMM and the fp32 CUDA-core GEMM vs a torch
fp32 reference of the same op, plus batch invariance (row results do not
depend on M)."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu

EPI_STORE, EPI_RESID, EPI_SWIGLU, EPI_F32 = 0, 1, 2, 3


def sr_gemm(A, W, C, epi, bias=None, bn=0):
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    dtype = 1 if A.dtype == torch.bfloat16 else 0
    M, K = A.shape
    N = W.shape[0]
    _native.check(lib.sr_gemm(dtype, M, N, K, A.data_ptr(), A.stride(0), W.data_ptr(),
                              W.stride(0), C.data_ptr(), C.stride(0), epi,
                              bias.data_ptr() if bias is not None else None, bn, None,
                              _native.stream_handle()), "sr_gemm")
    torch.cuda.synchronize()


def ref(A, W, bias=None):
    out = A.float() @ W.float().t()
    return out + bias if bias is not None else out


def swiglu_ref(acc):
    M, N = acc.shape
    blocks = acc.view(M, N // 32, 2, 16)
    g, u = blocks[:, :, 0, :], blocks[:, :, 1, :]
    return (torch.nn.functional.silu(g) * u).reshape(M, N // 2)


SHAPES = [(1, 128, 64), (5, 256, 128), (127, 384, 192), (128, 256, 1536),
          (300, 1536, 1536), (1280, 2048, 1536), (77, 1000, 96), (640, 512, 8960)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("bn", [128, 256])
def test_bf16_store_and_f32(M, N, K, bn):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    exp = ref(A, W, bias)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    sr_gemm(A, W, C, EPI_STORE, bias, bn)
    torch.testing.assert_close(C.float(), exp, rtol=1e-2, atol=1e-2)
    C32 = torch.empty(M, N, device="cuda", dtype=torch.float32)
    sr_gemm(A, W, C32, EPI_F32, bias, bn)
    torch.testing.assert_close(C32, exp, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M,N,K", [(5, 256, 128), (300, 1536, 1536), (1280, 1536, 8960)])
def test_bf16_residual_and_swiglu(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    R = torch.randn(M, N, device="cuda", generator=g)
    C = R.clone()
    sr_gemm(A, W, C, EPI_RESID)
    torch.testing.assert_close(C, R + ref(A, W), rtol=1e-4, atol=1e-3)
    S = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
    sr_gemm(A, W, S, EPI_SWIGLU)
    torch.testing.assert_close(S.float(), swiglu_ref(ref(A, W)), rtol=1e-2, atol=1e-2)


def test_bf16_batch_invariance():
    # rows computed inside M=1280 are bit-identical to the same rows at M=5
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(1280, 1536, device="cuda", generator=g).bfloat16()
    W = (torch.randn(2048, 1536, device="cuda", generator=g) * 0.05).bfloat16()
    big = torch.empty(1280, 2048, device="cuda", dtype=torch.float32)
    sr_gemm(A, W, big, EPI_F32)
    for start in (0, 3, 640, 1275):
        small = torch.empty(5, 2048, device="cuda", dtype=torch.float32)
        sr_gemm(A[start:start + 5].contiguous(), W, small, EPI_F32)
        assert torch.equal(small, big[start:start + 5])


@pytest.mark.parametrize("M,N,K", [(1, 64, 32), (37, 200, 128), (128, 384, 96)])
def test_f32_gemm(M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.randn(M, K, device="cuda", generator=g)
    W = torch.randn(N, K, device="cuda", generator=g) * 0.1
    bias = torch.randn(N, device="cuda", generator=g)
    exp = A.double() @ W.double().t()
    C = torch.empty(M, N, device="cuda")
    sr_gemm(A, W, C, EPI_STORE, bias)
    torch.testing.assert_close(C.double(), exp + bias.double(), rtol=1e-5, atol=1e-5)
    R = torch.randn(M, N, device="cuda", generator=g)
    C = R.clone()
    sr_gemm(A, W, C, EPI_RESID)
    torch.testing.assert_close(C.double(), R.double() + exp, rtol=1e-5, atol=1e-5)
    if N % 32 == 0:
        S = torch.empty(M, N // 2, device="cuda")
        sr_gemm(A, W, S, EPI_SWIGLU)
        torch.testing.assert_close(S.double(), swiglu_ref(exp), rtol=1e-5, atol=1e-5)


PAIR_CASES = [(1280, 1536, 1536, -112), (1280, 2048, 1536, -160), (300, 1000, 192, -112),
              (77, 512, 8960, -128), (1280, 17920, 1536, -256), (513, 3000, 640, -96),
              (256, 4096, 256, -224), (1000, 768, 896, -64), (1280, 1536, 8960, -192),
              # wide (> 128) residual tiles with ragged rows / a partial last tile
              (300, 1000, 192, -256), (77, 3584, 640, -192),
              # two pairs per cluster, A multicast (-(1024 + width)); odd tile counts included
              (1280, 1536, 8960, -1152), (1280, 2048, 1536, -1184), (300, 1000, 192, -1136),
              (77, 512, 8960, -1152), (1280, 17920, 1536, -1280), (1000, 768, 896, -1088)]


def tile_width(bn):
    w = -bn if bn < 0 else bn
    return w - 1024 if w > 1024 else w


@pytest.mark.parametrize("M,N,K,bn", PAIR_CASES)
def test_bf16_pair_kernel(M, N, K, bn):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    exp = ref(A, W, bias)
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    sr_gemm(A, W, C, EPI_STORE, bias, bn)
    torch.testing.assert_close(C.float(), exp, rtol=1e-2, atol=1e-2)
    C32 = torch.empty(M, N, device="cuda")
    sr_gemm(A, W, C32, EPI_F32, bias, bn)
    torch.testing.assert_close(C32, exp, rtol=1e-4, atol=1e-3)
    R = torch.randn(M, N, device="cuda", generator=g)
    C = R.clone()
    sr_gemm(A, W, C, EPI_RESID, None, bn)
    torch.testing.assert_close(C, R + ref(A, W), rtol=1e-4, atol=1e-3)
    if N % 32 == 0 and tile_width(bn) % 32 == 0:
        S = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        sr_gemm(A, W, S, EPI_SWIGLU, None, bn)
        torch.testing.assert_close(S.float(), swiglu_ref(ref(A, W)), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("bn", [-256, -112, 128, 256, -1280, -1136])
def test_argmax_epilogue(bn):
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    M, N, K = 300, 151936, 256
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    width = tile_width(bn)
    tiles = (N + width - 1) // width
    pv = torch.empty(M, tiles, device="cuda")
    pi = torch.empty(M, tiles, device="cuda", dtype=torch.int32)
    _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, pv.data_ptr(), tiles, 4, None, bn,
                              pi.data_ptr(), _native.stream_handle()), "sr_gemm argmax")
    torch.cuda.synchronize()
    logits = torch.empty(M, N, device="cuda")
    sr_gemm(A, W, logits, EPI_F32, None, bn)
    best = pv.max(1)
    idx = pi.gather(1, best.indices[:, None])[:, 0]
    assert torch.equal(idx.long(), logits.argmax(1))
    assert torch.equal(best.values, logits.max(1).values)


@pytest.mark.parametrize("bn", [-112, -1152])
def test_pair_batch_invariance(bn):
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(1280, 1536, device="cuda", generator=g).bfloat16()
    W = (torch.randn(1536, 1536, device="cuda", generator=g) * 0.05).bfloat16()
    big = torch.empty(1280, 1536, device="cuda")
    sr_gemm(A, W, big, EPI_F32, None, bn)
    for start in (0, 5, 256, 1275):
        small = torch.empty(5, 1536, device="cuda")
        sr_gemm(A[start:start + 5].contiguous(), W, small, EPI_F32, None, bn)
        assert torch.equal(small, big[start:start + 5])
    # the multicast cluster computes exactly what the single pair computes
    other = torch.empty(1280, 1536, device="cuda")
    sr_gemm(A, W, other, EPI_F32, None, -128 if bn == -1152 else -1136)
    assert torch.equal(other, big)


# Small-M ("swap") mode: live rows <= 128 run C^T = W A^T with K split into
# ranges summed in order; the large-M pair mode sums per-range TMEM
# accumulators in the same order.  Rows must come out bit-identical whichever
# mode (and however many rows) a launch runs, and match torch within bf16
# tolerance.  Shapes: 1.5B qkv/o/down, 0.5B down, ragged N and K.
SWAP_SHAPES = [(512, 256), (1536, 1536), (2048, 1536), (1536, 8960), (896, 4864), (1000, 448), (4608, 3584)]


@pytest.fixture
def swap_everywhere():
    """Small-M mode for every swap-capable plan at <= 128 live rows (the
    default threshold depends on the weight bytes)."""
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    _native.check(lib.sr_set_gemm_swap_max_m(128), "swap threshold")
    yield
    _native.check(lib.sr_set_gemm_swap_max_m(-1), "swap threshold")


@pytest.mark.parametrize("N,K", SWAP_SHAPES)
def test_small_m_mode_bit_identical_to_pair_mode(N, K, swap_everywhere):
    from paper_2511_16193_b200 import _native

    splits = _native.lib().sr_gemm_splits(N, K, EPI_F32)
    assert splits >= 1
    if (N, K) == (1536, 8960):
        assert splits > 1  # the K-range reduction is exercised
    g = torch.Generator(device="cuda").manual_seed(N + 3 * K)
    big_m = 320
    A = torch.randn(big_m, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    R0 = torch.randn(big_m, N, device="cuda", generator=g)
    exp = ref(A, W, bias)
    for epi in (EPI_F32, EPI_STORE, EPI_RESID, EPI_SWIGLU):
        if epi == EPI_SWIGLU and N % 32 != 0:
            continue
        out_dtype = torch.bfloat16 if epi in (EPI_STORE, EPI_SWIGLU) else torch.float32
        b = None if epi in (EPI_RESID, EPI_SWIGLU) else bias
        ncols = N // 2 if epi == EPI_SWIGLU else N
        big = R0.clone() if epi == EPI_RESID else torch.empty(big_m, ncols, device="cuda", dtype=out_dtype)
        sr_gemm(A, W, big, epi, b)
        for m in (1, 17, 32, 64, 100, 128):
            small = R0[:m].clone() if epi == EPI_RESID else torch.empty(m, ncols, device="cuda", dtype=out_dtype)
            sr_gemm(A[:m].contiguous(), W, small, epi, b)
            assert torch.equal(small, big[:m]), f"epi {epi} m {m}: small-M mode differs from the pair mode"
        if epi == EPI_F32:
            torch.testing.assert_close(big, exp, rtol=1e-4, atol=2e-3)
        if epi == EPI_RESID:
            torch.testing.assert_close(big, R0 + ref(A, W), rtol=1e-4, atol=2e-3)
        if epi == EPI_SWIGLU:
            torch.testing.assert_close(big.float(), swiglu_ref(ref(A, W)), rtol=2e-2, atol=2e-2)


def test_small_m_mode_repeated_launches_reset_counters(swap_everywhere):
    """The K-range arrival counters reset themselves: many back-to-back small-M
    launches (different row counts) give the same bits as the first."""
    N, K = 1536, 8960
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(128, K, device="cuda", generator=g).bfloat16()
    W = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
    first = torch.empty(128, N, device="cuda")
    sr_gemm(A, W, first, EPI_F32)
    for it in range(20):
        m = 1 + (it * 37) % 128
        out = torch.empty(m, N, device="cuda")
        sr_gemm(A[:m].contiguous(), W, out, EPI_F32)
        assert torch.equal(out, first[:m])
