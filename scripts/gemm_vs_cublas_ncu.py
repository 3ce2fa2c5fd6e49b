"""Launch the down-projection GEMM (M=1280, N=1536, K=8960) through our pair
kernel and through cuBLAS (torch) once each, for a side-by-side ncu capture."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_16193_b200 import _native  # noqa: E402

lib = _native.lib()
st = _native.stream_handle()
M, N, K = 1280, 1536, 8960
A = torch.randn(M, K, device="cuda").bfloat16()
W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
C = torch.zeros(M, N, device="cuda")
for bn in [int(x) for x in (sys.argv[1:] or ["-128"])]:
    _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), N, 1,
                              None, bn, None, st), "down")
torch.matmul(A, W.t())
torch.cuda.synchronize()
print("ok")
