import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2511_16193_b200 import _native
lib = _native.lib(); st = _native.stream_handle()
M = 1280
def t(f, it=30):
    for _ in range(3): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(it): f()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / it * 1e3
for name, N, K in (("down", 1536, 8960), ("o", 1536, 1536), ("qkv", 2048, 1536)):
    A = torch.randn(M, K, device="cuda").bfloat16(); W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    C = torch.zeros(M, N, device="cuda")
    for bn in (-96, -112, -128, -1136, -1152, -160, -1184):
        us = t(lambda: lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), N, 1, None, bn, None, st))
        print(f"{name} bn={bn}: {us:.1f} us")
