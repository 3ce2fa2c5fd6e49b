"""Small workload that launches every kernel family of the library once or a
few times (for compute-sanitizer memcheck / racecheck / synccheck runs):
tiny target in bf16 and fp32, n-gram + model drafters with Best-of-N,
compaction, keyed sampling, rejection sampling, the host-facing step,
decoupled rounds, and the truth-mode simulate.

    compute-sanitizer --tool memcheck python scripts/sanitize_workload.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200 import scenarios  # noqa: E402
from paper_2511_16193_b200.decoupled import run_local  # noqa: E402
from paper_2511_16193_b200.engine import ModelDrafter, NgramDrafter, RolloutEngine, SyntheticDrafter  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402
from paper_2511_16193_b200.sim import SimConfig, simulate  # noqa: E402
from paper_2511_16193_b200.workload import gen_trace  # noqa: E402


def main():
    s = shape("tiny")
    w = init_weights(s, seed=0)
    rng = np.random.default_rng(0)
    words = rng.integers(0, s.vocab, 12)
    B, k = 4, 4
    prompts = [words[rng.integers(0, 12, int(rng.integers(20, 70)))].astype(np.int32) for _ in range(B)]
    max_new = [20, 9, 14, 3]
    for dtype in ("bf16", "fp32"):
        m = DeviceModel(s, w, dtype=dtype, max_requests=B, max_len=160, max_tokens=B * 3 * (k + 2),
                        max_seqs=B * 3, branches=B * 2, logits_capacity=B * 3 * (k + 2))
        d = DeviceModel(s, w, dtype=dtype, max_requests=B, max_len=160, max_tokens=B * (k + 2), max_seqs=B,
                        logits_capacity=B * (k + 2))
        for temp in (0.0, 1.0):
            eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(NgramDrafter(), ModelDrafter(d), NgramDrafter(2, 3)),
                                history=64, temperature=temp, seed=3)
            eng.prefill()
            eng.run()
        eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(ModelDrafter(d),), history=64, temperature=1.0,
                            seed=3, acceptance="rejection")
        eng.prefill()
        eng.run()
        print(dtype, "engine ok", flush=True)
    m = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=160, max_tokens=B * (k + 1), max_seqs=B)
    eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(NgramDrafter(),), history=1)
    eng.prefill()
    budget = torch.tensor(max_new, dtype=torch.int32).pin_memory()
    res = torch.zeros((B, 4 + k + 2), dtype=torch.int32).pin_memory()
    g = eng.capture_io(budget, res)
    for _ in range(6):
        eng.step_io(g)
    torch.cuda.synchronize()
    plain = RolloutEngine(m, prompts, max_new, k=0, history=1)
    plain.prefill()
    plain.run()
    trace = gen_trace(scenarios.default_trace_spec(batch=B, seed=0))
    run_local(m, prompts, max_new, k, SyntheticDrafter(plain.outputs(), trace, "ngram", 0, vocab=s.vocab), graphs=False)
    print("decoupled ok", flush=True)
    cfg = SimConfig(trace=gen_trace(scenarios.default_trace_spec(batch=4, seed=0)), model=scenarios.default_cost_model(),
                    policy="decoupled", method=scenarios.DEFAULT_METHOD, seed=0,
                    scale_cost=scenarios.default_scale_cost(), estimator_priors=scenarios.estimator_priors())
    simulate(cfg)
    torch.cuda.synchronize()
    print("sanitize workload done", flush=True)


if __name__ == "__main__":
    main()
