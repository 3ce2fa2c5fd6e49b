"""One GEMM shape launched a few times (ncu target).
    python scripts/gemm_one.py N K M [epi]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_16193_b200 import _native  # noqa: E402

N, K, M = (int(x) for x in sys.argv[1:4])
epi = int(sys.argv[4]) if len(sys.argv) > 4 else 3
lib = _native.lib()
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
A = torch.randn(M, K, device="cuda").bfloat16()
C = torch.zeros(M, N, device="cuda")
for _ in range(5):
    _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), N, epi, None, 0, None,
                              _native.stream_handle()), "gemm")
torch.cuda.synchronize()
print("ok", N, K, M, "splits", lib.sr_gemm_splits(N, K, epi))
