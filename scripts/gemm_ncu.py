"""Launch the verify GEMMs once per tile config (for ncu)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2511_16193_b200 import _native  # noqa: E402

lib = _native.lib()
st = _native.stream_handle()
M = 1280
for name, N, K, epi, bns in (("gate_up", 17920, 1536, 2, (256, -256)), ("down", 1536, 8960, 1, (128, -112, -256))):
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    C = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.bfloat16 if epi == 2 else torch.float32)
    for bn in bns:
        for _ in range(2):
            _native.check(lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), C.stride(0), epi,
                                      None, bn, None, st), name)
torch.cuda.synchronize()
print("ok")
