"""Down / gate_up / o / qkv GEMMs timed (a) back to back, (b) each after an
L2 flush (cold weights), (c) each after a device sync (no launch overlap) --
separates cold-weight cost from launch overlap in the in-step numbers."""
import sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2511_16193_b200 import _native
lib = _native.lib(); st = _native.stream_handle()
M = 1280
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for name, N, K, epi in (("qkv", 2048, 1536, 0), ("o", 1536, 1536, 1), ("gate_up", 17920, 1536, 2), ("down", 1536, 8960, 1)):
    A = torch.randn(M, K, device="cuda").bfloat16(); W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    C = torch.zeros(M, N // 2 if epi == 2 else N, device="cuda", dtype=torch.bfloat16 if epi in (0, 2) else torch.float32)
    f = lambda: lib.sr_gemm(1, M, N, K, A.data_ptr(), K, W.data_ptr(), K, C.data_ptr(), C.stride(0), epi, None, 0, None, st)
    for _ in range(3): f()
    torch.cuda.synchronize()
    res = {}
    for mode in ("back2back", "cold", "synced"):
        ts = []
        for it in range(10):
            if mode == "cold":
                flush.fill_(it)
            if mode != "back2back":
                torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(); f(); e.record()
            if mode != "back2back":
                torch.cuda.synchronize()
            ts.append((s, e))
        torch.cuda.synchronize()
        res[mode] = sorted(s.elapsed_time(e) * 1e3 for s, e in ts)[5]
    print(name, {k: round(v, 1) for k, v in res.items()})
