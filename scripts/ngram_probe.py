"""Time the n-gram drafter kernel (K4) on large batched contexts: HBM GB/s
over the context tokens it must scan.

    python scripts/ngram_probe.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_16193_b200 import _native  # noqa: E402


def main():
    lib = _native.lib()
    st = _native.stream_handle()
    for B, L in ((256, 1600), (256, 8192), (1024, 4096), (256, 32768)):
        g = torch.Generator(device="cuda").manual_seed(0)
        tokens = torch.randint(0, 50, (B, L + 64), generator=g, device="cuda", dtype=torch.int32)
        lens = torch.full((B,), L, dtype=torch.int32, device="cuda")
        drafts = torch.empty((B, 4), dtype=torch.int32, device="cuda")
        nd = torch.empty(B, dtype=torch.int32, device="cuda")
        scratch = torch.zeros(2 * B, dtype=torch.int64, device="cuda")

        def go():
            _native.check(lib.sr_ngram_propose(B, tokens.data_ptr(), L + 64, lens.data_ptr(), 1, 3, 4,
                                               drafts.data_ptr(), nd.data_ptr(), scratch.data_ptr(), st), "ngram")
        for _ in range(3):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            go()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"B={B} ctx={L}: {us:8.1f} us  {B * L * 4 / us / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main()
