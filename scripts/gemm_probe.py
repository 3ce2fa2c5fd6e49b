"""Time the tcgen05 GEMM on the verify-forward shapes against cuBLAS (torch).

    python scripts/gemm_probe.py [--m 1280]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200 import _native  # noqa: E402

SHAPES_15B = {  # name: (N, K, epilogue)
    "qkv": (2048, 1536, 0), "o": (1536, 1536, 1), "gate_up": (17920, 1536, 2),
    "down": (1536, 8960, 1), "lm_head": (151936, 1536, 3),
}
SHAPES_32B = {
    "qkv": (7168, 5120, 0), "o": (5120, 5120, 1), "gate_up": (55296, 5120, 2),
    "down": (5120, 27648, 1),
}
SHAPES_7B = {
    "qkv": (4608, 3584, 0), "o": (3584, 3584, 1), "gate_up": (37888, 3584, 2),
    "down": (3584, 18944, 1),
}


def time_it(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1280)
    ap.add_argument("--model", choices=["1.5b", "7b", "32b"], default="1.5b")
    ap.add_argument("--only", default=None, help="comma-separated GEMM names")
    ap.add_argument("--bns", type=int, nargs="+", default=[128, 256, -128, -160, -192, -256, -1152, -1184, 0],
                    help="tile widths: >0 single-CTA, <0 CTA pair, <-1024 pair + A multicast, 0 auto")
    args = ap.parse_args()
    lib = _native.lib()
    M = args.m
    st = _native.stream_handle()
    shapes = {"7b": SHAPES_7B, "32b": SHAPES_32B}.get(args.model, SHAPES_15B)
    for name, (N, K, epi) in shapes.items():
        if args.only and name not in args.only.split(","):
            continue
        A = torch.randn(M, K, device="cuda").bfloat16()
        W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
        if epi == 1:
            C = torch.zeros(M, N, device="cuda")
        elif epi == 2:
            C = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        elif epi == 3:
            C = torch.empty(M, N, device="cuda")
        else:
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for bn in args.bns:
            if False:
                continue

            def run():
                _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K,
                                          C.data_ptr(), C.stride(0), epi, None, bn, None, st), "gemm")
            ms = time_it(run)
            tf = 2 * M * N * K / ms / 1e9
            print(f"{name:8s} M={M} N={N} K={K} bn={bn}: {ms*1e3:8.1f} us  {tf:7.1f} TFLOP/s")
        ms = time_it(lambda: torch.matmul(A, W.t()))
        print(f"{name:8s} cuBLAS: {ms*1e3:8.1f} us  {2*M*N*K/ms/1e9:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()
