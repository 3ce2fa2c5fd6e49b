"""Short, profiler-friendly run of the bench workload's speculation step
(1.5B-shaped target, 256 prompts, k=4 windows): prefill, then --steps steps.

    ncu --profile-from-start off --set full -k regex:attn_bf16 -c 2 python scripts/profile_step.py
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200 import scenarios  # noqa: E402
from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402
from paper_2511_16193_b200.streams import stream  # noqa: E402
from paper_2511_16193_b200.workload import gen_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--model", default="qwen2.5-1.5b")
    a = ap.parse_args()
    s = shape(a.model)
    trace = gen_trace(scenarios.default_trace_spec(batch=a.batch, seed=0))
    prompts = [stream(0, r.id, "prompt").integers(0, s.vocab, size=r.prompt_len).astype(np.int32)
               for r in trace]
    budget = [64] * a.batch
    m = DeviceModel(s, init_weights(s, seed=0, device="cuda"), dtype="bf16", max_requests=a.batch,
                    max_len=1024 + 80, max_tokens=a.batch * 5, max_seqs=a.batch)
    truth = [list(np.random.default_rng(i).integers(0, s.vocab, size=64)) for i in range(a.batch)]
    eng = RolloutEngine(m, prompts, budget, k=4, drafters=(SyntheticDrafter(truth, trace, "draft-0.5b", 0),),
                        bonus_token=True, history=1)
    eng.prefill()
    eng.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off
    for _ in range(a.steps):
        eng.step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("ok")


if __name__ == "__main__":
    main()
