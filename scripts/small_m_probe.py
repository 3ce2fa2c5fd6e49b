"""Decode-step latency at small batch (the HBM-bound small-M regime of
drafters, plain decode and tail windows): one forward of B single-token rows
over ~600-token contexts, CUDA-graph replay, CUDA events.  Roofline =
(weights + KV bytes) / HBM peak.  (A split-K mma.sync "narrow" path was
measured against this and rejected: branch narrow-smallm-experiment.)

    python scripts/small_m_probe.py
"""
from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2511_16193_b200.model import DeviceModel, init_weights, seq_table, shape  # noqa: E402


def hbm_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    return json.loads(f.read_text())["hbm_gbs"] if f.exists() else 6550.0


def probe(name, B, ctx=600, reps=20):
    s = shape(name)
    w = init_weights(s, seed=0, device="cuda")
    res = {}
    for narrow in (0,):
        m = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=ctx + 64, max_tokens=max(B * (ctx + 1), 64),
                        max_seqs=B)
        rng = np.random.default_rng(0)
        toks = torch.from_numpy(rng.integers(0, s.vocab, (B, ctx + 1)).astype(np.int32)).cuda()
        rows = [(b * ctx, ctx, b, 0, -1) for b in range(B)]
        m.forward(toks[:, :ctx].reshape(-1).contiguous(),
                  torch.arange(ctx, dtype=torch.int32, device="cuda").repeat(B), seq_table(rows, "cuda"),
                  num_seqs=B, max_q_len=ctx, max_key=ctx - 1, out=torch.empty(B * ctx, dtype=torch.int32,
                                                                                 device="cuda"))
        ids, pos = toks[:, ctx].contiguous(), torch.full((B,), ctx, dtype=torch.int32, device="cuda")
        seqs = seq_table([(b, 1, b, ctx, -1) for b in range(B)], "cuda")
        out = torch.empty(B, dtype=torch.int32, device="cuda")

        def step():
            m.forward(ids, pos, seqs, num_seqs=B, max_q_len=1, max_key=ctx, out=out)
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
        if os.environ.get("SR_PROFILE_STEP"):
            torch.cuda.synchronize()
            torch.cuda.profiler.start()
            g.replay()
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res["narrow" if narrow else "wide"] = ms
        del m, g
        torch.cuda.empty_cache()
    wbytes = 2 * (s.linear_params() + (0 if s.tied else 0))
    kv = B * ctx * s.kv_bytes_per_token()
    roof_ms = (wbytes + kv) / (hbm_peak() * 1e9) * 1e3
    return {"model": name, "batch": B, "ctx": ctx, "ms": round(res["wide"], 3), "roofline_ms": round(roof_ms, 3),
            "frac": round(roof_ms / res["wide"], 3)}


if __name__ == "__main__":
    models = sys.argv[1].split(",") if len(sys.argv) > 1 else ["qwen2.5-0.5b", "qwen2.5-1.5b"]
    batches = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [32, 64]
    for name in models:
        for B in batches:
            print(json.dumps(probe(name, B)), flush=True)
