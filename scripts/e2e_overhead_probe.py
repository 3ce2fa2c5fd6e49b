"""Where the host-facing step's time goes: the same speculation step replayed
(a) as the installed step graph, (b) as the capture_io graph (H2D budgets,
step, result pack, D2H) back to back, (c) as the bench's e2e loop (host
reads step i-1 while step i runs).  1.5B target, 256 prompts, k = 4, n-gram
drafter, CUDA events.

    python scripts/e2e_overhead_probe.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402


def main(steps=40):
    s = shape("qwen2.5-1.5b")
    B, K = 256, 4
    rng = np.random.default_rng(0)
    prompts = [rng.integers(0, s.vocab, int(n)).astype(np.int32) for n in rng.integers(128, 1025, B)]
    budget = [4 * (steps * 3 + 20)] * B
    m = DeviceModel(s, init_weights(s, seed=0, device="cuda"), dtype="bf16", max_requests=B,
                    max_len=max(len(p) for p in prompts) + budget[0] + 16, max_tokens=B * (K + 1), max_seqs=B)
    eng = RolloutEngine(m, prompts, budget, k=K, drafters=(NgramDrafter(1, 3),), bonus_token=True, history=1)
    eng.prefill()
    eng.capture()
    st = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn(steps)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    out = {"step_graph_ms": timed(lambda n=1: [eng.step() for _ in range(n)])}
    bh = torch.tensor(budget, dtype=torch.int32).pin_memory()
    res = [torch.empty((B, 4 + K + 2), dtype=torch.int32).pin_memory() for _ in range(2)]
    graphs = [eng.capture_io(bh, r) for r in res]
    out["io_graph_back_to_back_ms"] = timed(lambda n=1: [eng.step_io(graphs[i % 2]) for i in range(n)])
    out["io_graph_same_graph_ms"] = timed(lambda n=1: [eng.step_io(graphs[0]) for i in range(n)])
    g2 = [eng.capture(install=False) for _ in range(2)]
    out["step_graph_alternating_ms"] = timed(lambda n=1: [g2[i % 2].replay() for i in range(n)])
    done = [torch.cuda.Event(), torch.cuda.Event()]

    def loop(n=1):
        for i in range(n):
            eng.step_io(graphs[i % 2])
            done[i % 2].record(st)
            if i > 0:
                done[(i - 1) % 2].synchronize()
                int(res[(i - 1) % 2][0, 2])
        done[(n - 1) % 2].synchronize()
    out["e2e_loop_ms"] = timed(loop)
    print(json.dumps({k: round(v, 4) for k, v in out.items()}))


if __name__ == "__main__":
    main()
