"""List the cuBLAS kernels (name, grid, block, duration) torch picks for the
verify-forward GEMM shapes -- the tile/cluster choices we compare against."""
import json
import torch
from torch.profiler import profile, ProfilerActivity

SHAPES = {"qkv": (2048, 1536), "o": (1536, 1536), "gate_up": (17920, 1536), "down": (1536, 8960)}
M = 1280
for name, (N, K) in SHAPES.items():
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    for _ in range(3):
        torch.matmul(A, W.t())
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            torch.matmul(A, W.t())
        torch.cuda.synchronize()
    prof.export_chrome_trace("/tmp/t.json")
    ev = [e for e in json.load(open("/tmp/t.json"))["traceEvents"] if e.get("cat") == "kernel"]
    for e in ev[-2:]:
        a = e["args"]
        print(name, e["name"][:120], "grid", a.get("grid"), "block", a.get("block"),
              "smem", a.get("shared memory"), "regs", a.get("registers per thread"), "dur_us", e["dur"])
