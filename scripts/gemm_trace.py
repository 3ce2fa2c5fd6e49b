"""Per-CTA phase timeline of one GEMM launch (measurement build with
-DSR_GEMM_TRACE, loaded from build/trace/): %globaltimer stamps of entry,
griddepcontrol.wait done, first operands, first accumulator ready,
partials/counter done, epilogue done, exit.

    SR_EXTRA_NVCC_FLAGS=-DSR_GEMM_TRACE python scripts/gemm_trace.py --build
    python scripts/gemm_trace.py --n 1536 --k 8960 --m 32 64 128
"""
from __future__ import annotations

import argparse
import ctypes
import os
import shutil
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
TRACE_LIB = ROOT / "scripts" / "_trace" / "libspecrollout_b200_trace.so"  # travels to the GPU box
EVENTS = ["entry", "wait_done", "first_stage", "acc_ready", "counter", "epi_done", "exit", "g0_loaded"]


def build_trace():
    from paper_2511_16193_b200 import build

    os.environ["SR_EXTRA_NVCC_FLAGS"] = "-DSR_GEMM_TRACE"
    build.FLAGS.append("-DSR_GEMM_TRACE")
    lib = build.build()
    TRACE_LIB.parent.mkdir(parents=True, exist_ok=True)
    shutil.copy(lib, TRACE_LIB)
    build.FLAGS.remove("-DSR_GEMM_TRACE")
    (build.OBJ / "link.stamp").unlink(missing_ok=True)
    build.build()  # restore the release library
    print("trace library:", TRACE_LIB)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    ap.add_argument("--n", type=int, default=1536)
    ap.add_argument("--k", type=int, default=8960)
    ap.add_argument("--m", type=int, nargs="+", default=[32, 128])
    ap.add_argument("--epi", type=int, default=3)
    args = ap.parse_args()
    if args.build:
        build_trace()
        return
    import torch

    from paper_2511_16193_b200 import _native

    lib = _native.load(TRACE_LIB)
    N, K = args.n, args.k
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    print(f"N={N} K={K} splits={lib.sr_gemm_splits(N, K, args.epi)}")
    for M in args.m:
        A = torch.randn(M, K, device="cuda").bfloat16()
        C = torch.zeros(M, N, device="cuda")
        for it in range(3):
            if it == 2:
                torch.cuda.synchronize()
                lib.sr_debug_gemm_trace(None, 0)
            _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), N, args.epi,
                                      None, 0, None, _native.stream_handle()), "gemm")
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (1024 * 8))()
        lib.sr_debug_gemm_trace(buf, 1024 * 8)
        rows = []
        for b in range(1024):
            ev = [buf[b * 8 + e] for e in range(8)]
            if ev[0] == 0:
                continue
            rows.append((b, ev))
        t0 = min(ev[0] for _, ev in rows)
        print(f"M={M}: {len(rows)} CTAs; times in us from the first entry")
        for b, ev in rows[:: max(1, len(rows) // 12)]:
            print(f"  cta {b:4d} " + " ".join(f"{n}={(e - t0) / 1e3:7.2f}" if e else f"{n}=   -   "
                                              for n, e in zip(EVENTS, ev)))
        last = max(ev[6] for _, ev in rows)
        print(f"  span {(last - t0) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
