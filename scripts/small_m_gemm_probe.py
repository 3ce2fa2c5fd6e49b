"""Small-M GEMM probe: per-launch time of the tcgen05 GEMM variants at live M
<= 128 (graph of back-to-back launches, warm L2 excluded by weights > L2 for
the big shapes), weight-stream GB/s against HBM peak, cuBLAS beside it, and
whether the variants produce bit-identical fp32 results (the batch-invariance
question for a small-M path).

    python scripts/small_m_gemm_probe.py [--model 32b] [--m 32 64 128]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200 import _native  # noqa: E402

SHAPES = {
    "0.5b": {"qkv": (1152, 896), "o": (896, 896), "gate_up": (9728, 896), "down": (896, 4864)},
    "1.5b": {"qkv": (2048, 1536), "o": (1536, 1536), "gate_up": (17920, 1536), "down": (1536, 8960)},
    "7b": {"qkv": (4608, 3584), "o": (3584, 3584), "gate_up": (37888, 3584), "down": (3584, 18944)},
    "32b": {"qkv": (7168, 5120), "o": (5120, 5120), "gate_up": (55296, 5120), "down": (5120, 27648)},
}


def graph_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        g.capture_begin()
        for _ in range(reps):
            fn(st)
        g.capture_end()
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (3 * reps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", nargs="+", default=["0.5b", "7b", "32b"])
    ap.add_argument("--m", type=int, nargs="+", default=[32, 64, 128])
    ap.add_argument("--bns", type=int, nargs="+", default=[0, 128, 256, -256, -128, -64])
    args = ap.parse_args()
    lib = _native.lib()
    peak = 6550.7
    for model in args.model:
        for name, (N, K) in SHAPES[model].items():
            W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
            # several weight copies so consecutive launches do not hit L2
            copies = max(1, int(300e6 // (N * K * 2)))
            Ws = [W.clone() for _ in range(copies)]
            for M in args.m:
                A = torch.randn(M, K, device="cuda").bfloat16()
                C = torch.zeros(M, N, device="cuda")
                ref = None
                line = []
                for bn in args.bns:
                    idx = [0]

                    def run(st=None, bn=bn):
                        w = Ws[idx[0] % copies]
                        idx[0] += 1
                        h = _native.stream_handle(st) if st is not None else _native.stream_handle()
                        _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, w.data_ptr(), K, C.data_ptr(), N,
                                                  3, None, bn, None, h), "gemm")
                    try:
                        ms = graph_time(run)
                    except Exception as e:  # noqa: BLE001
                        line.append(f"bn={bn}: err {e}")
                        continue
                    C.zero_()
                    run()
                    torch.cuda.synchronize()
                    same = None
                    if ref is None:
                        ref = C.clone()
                    else:
                        same = bool(torch.equal(C, ref))
                    gbs = N * K * 2 / (ms * 1e-3) / 1e9
                    line.append(f"bn={bn}: {ms*1e3:7.1f}us {gbs:6.0f}GB/s({gbs/peak:.2f}){'' if same is None else (' =' if same else ' DIFF')}")
                Af = A
                ms = graph_time(lambda st=None: torch.matmul(Af, Ws[0].t()))
                gbs = N * K * 2 / (ms * 1e-3) / 1e9
                line.append(f"cuBLAS {ms*1e3:7.1f}us {gbs:6.0f}GB/s")
                print(f"{model:5s} {name:8s} M={M:4d} N={N:6d} K={K:6d} | " + " | ".join(line), flush=True)
            del Ws, W
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
