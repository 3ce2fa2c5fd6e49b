"""Gap between consecutive replays of the step graph (CUPTI kernel
timestamps): the last kernel's end of replay i to the first kernel's start of
replay i+1, and each replay's span.  1.5B, 256 prompts, k = 4, n-gram drafter.

    python scripts/replay_gap_probe.py
"""
from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402


def main(reps=6):
    from torch.profiler import ProfilerActivity, profile

    s = shape(os.environ.get("MODEL", "qwen2.5-1.5b"))
    B, K = 256, 4
    rng = np.random.default_rng(0)
    prompts = [rng.integers(0, s.vocab, int(n)).astype(np.int32) for n in rng.integers(128, 1025, B)]
    budget = [400] * B
    m = DeviceModel(s, init_weights(s, seed=0, device="cuda"), dtype="bf16", max_requests=B,
                    max_len=max(len(p) for p in prompts) + budget[0] + 16, max_tokens=B * (K + 1), max_seqs=B)
    eng = RolloutEngine(m, prompts, budget, k=K, drafters=(NgramDrafter(1, 3),), bonus_token=True, history=1)
    eng.prefill()
    eng.capture()
    for _ in range(3):
        eng.step()
    torch.cuda.synchronize()
    per = None
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            eng.step()
        torch.cuda.synchronize()
    path = tempfile.mktemp(suffix=".json")
    prof.export_chrome_trace(path)
    ev = sorted((e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"), key=lambda e: e["ts"])
    os.unlink(path)
    per = len(ev) // reps
    spans, gaps, firsts = [], [], []
    for r in range(reps):
        run = ev[r * per:(r + 1) * per]
        t0 = run[0]["ts"]
        t1 = max(e["ts"] + e["dur"] for e in run)
        spans.append(t1 - t0)
        if r:
            gaps.append(t0 - prev_end)
        prev_end = t1
        firsts.append(run[0]["name"][:40])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        eng.step()
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"kernels_per_replay": per, "span_us": [round(x, 1) for x in spans],
                      "gap_us": [round(x, 1) for x in gaps], "first_kernel": firsts[0],
                      "event_ms_per_step": round(e0.elapsed_time(e1) / 20, 4)}))


if __name__ == "__main__":
    main()
