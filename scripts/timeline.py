"""In-graph kernel timeline of one CUDA-graph replay (CUPTI through
torch.profiler): start/end of every kernel as the GPU ran it, PDL overlap
included.  Prints per-kernel-name totals of the span each kernel occupies
exclusively (gaps and overlaps resolved in launch order).

    python scripts/timeline.py decode qwen2.5-1.5b 32
    python scripts/timeline.py step            # bench workload (1.5B, 256 prompts)
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def decode_graph(name, B, ctx=600):
    import numpy as np

    from paper_2511_16193_b200.model import DeviceModel, init_weights, seq_table, shape

    s = shape(name)
    w = init_weights(s, seed=0, device="cuda")
    m = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=ctx + 64, max_tokens=max(B * (ctx + 1), 64),
                    max_seqs=B)
    rng = np.random.default_rng(0)
    toks = torch.from_numpy(rng.integers(0, s.vocab, (B, ctx + 1)).astype(np.int32)).cuda()
    rows = [(b * ctx, ctx, b, 0, -1) for b in range(B)]
    m.forward(toks[:, :ctx].reshape(-1).contiguous(), torch.arange(ctx, dtype=torch.int32, device="cuda").repeat(B),
              seq_table(rows, "cuda"), num_seqs=B, max_q_len=ctx, max_key=ctx - 1,
              out=torch.empty(B * ctx, dtype=torch.int32, device="cuda"))
    ids, pos = toks[:, ctx].contiguous(), torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    seqs = seq_table([(b, 1, b, ctx, -1) for b in range(B)], "cuda")
    out = torch.empty(B, dtype=torch.int32, device="cuda")

    def step():
        m.forward(ids, pos, seqs, num_seqs=B, max_q_len=1, max_key=ctx, out=out)
    return step, (m, w)




def timeline(step, reps=3):
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        g.capture_begin()
        step()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            g.replay()
        torch.cuda.synchronize()
    path = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
    os.unlink(path)
    ev.sort(key=lambda e: e["ts"])
    per = len(ev) // reps  # kernels per replay
    runs = [ev[i * per:(i + 1) * per] for i in range(reps)]
    run = runs[-1]
    t0 = run[0]["ts"]
    span = max(e["ts"] + e["dur"] for e in run) - t0
    excl = defaultdict(float)
    dur = defaultdict(float)
    cnt = defaultdict(int)
    end_prev = t0
    for e in run:
        nm = e["name"].replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][-60:]
        s, f = e["ts"], e["ts"] + e["dur"]
        excl[nm] += max(0.0, f - max(s, end_prev))  # time this kernel extends the timeline
        end_prev = max(end_prev, f)
        dur[nm] += e["dur"]
        cnt[nm] += 1
    print(f"kernels {len(run)}  span {span:.1f} us  (replays seen {len(runs)})")
    for nm in sorted(excl, key=lambda k: -excl[k])[:14]:
        print(f"  {excl[nm]:8.1f} us excl  {dur[nm]:8.1f} us busy  n={cnt[nm]:4d}  {nm}")
    if os.environ.get("TL_DUMP"):
        for e in run[: int(os.environ["TL_DUMP"])]:
            nm = e["name"].replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][-50:]
            print(f"    {e['ts'] - t0:9.1f} +{e['dur']:7.1f}  {nm}")
    return run


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "decode"
    if what == "decode":
        name = sys.argv[2] if len(sys.argv) > 2 else "qwen2.5-1.5b"
        B = int(sys.argv[3]) if len(sys.argv) > 3 else 32
        step, keep = decode_graph(name, B)
        timeline(step)
    if what == "trace":  # SR_LIB_PATH=scripts/_trace/libspecrollout_b200_trace.so: last small-M GEMM of a decode step
        import ctypes

        from paper_2511_16193_b200 import _native

        name = sys.argv[2] if len(sys.argv) > 2 else "qwen2.5-1.5b"
        B = int(sys.argv[3]) if len(sys.argv) > 3 else 32
        step, keep = decode_graph(name, B)
        lib = _native.lib()
        step()
        torch.cuda.synchronize()
        lib.sr_debug_gemm_trace(None, 0)
        step()
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (1024 * 8))()
        lib.sr_debug_gemm_trace(buf, 1024 * 8)
        names = ["entry", "wait", "stage0", "acc", "counter", "epi", "exit", "g0"]
        rows = [(b, [buf[b * 8 + e] for e in range(8)]) for b in range(1024) if buf[b * 8]]
        t0 = min(ev[0] for _, ev in rows)
        for b, ev in rows[:64]:
            print(f"cta {b:4d} " + " ".join(f"{n}={(x - t0) / 1e3:6.2f}" if x else f"{n}=   -  " for n, x in zip(names, ev)))
