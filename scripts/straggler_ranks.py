"""Prompt-sharded rollout to completion over N ranks with cross-rank
straggler pulls (reference ``sim.py:546-593``; ``straggler.StragglerPull``).

Each rank owns ``trace[rank::world]`` (``sim.py:307-309``), runs its shard
through ``policy.RolloutDriver`` with the reference-acceptance drafter over
the target's own greedy continuation, and -- with ``--pull`` -- drained ranks
adopt the slowest live requests of the busiest rank (token row, KV pages and
drafter rows over NCCL P2P).  Rank 0 prints one JSON line: makespan (max
over ranks of the device time to the last committing step), committed
tokens, moves, bytes moved, and whether every request's output equals plain
greedy decoding.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/straggler_ranks.py --pull
    torchrun --nproc-per-node 2 ... scripts/straggler_ranks.py --backend gloo  # both ranks on GPU 0
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2511_16193_b200 import scenarios  # noqa: E402
from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402
from paper_2511_16193_b200.policy import RolloutDriver  # noqa: E402
from paper_2511_16193_b200.straggler import StragglerPull  # noqa: E402
from paper_2511_16193_b200.streams import stream  # noqa: E402
from paper_2511_16193_b200.workload import gen_trace  # noqa: E402

K = 4


def skewed(trace, short: int):
    """Rank-0-heavy imbalance for tests: even-indexed requests (rank 0 of
    two) end after ``short`` tokens."""
    return [dataclasses.replace(r, true_len=min(r.true_len, short)) if i % 2 == 0 else r
            for i, r in enumerate(trace)]


def run(args) -> dict:
    rank, world = dist.get_rank(), dist.get_world_size()
    s = shape(args.model, args.layers)
    spec = scenarios.default_trace_spec(batch=args.batch, seed=0)
    spec = type(spec)(**{**spec.__dict__, "length_cap": args.cap})
    trace = gen_trace(spec)
    if args.skew:
        trace = skewed(trace, args.skew)
    prompts = {r.id: stream(0, r.id, "prompt").integers(0, s.vocab, size=min(r.prompt_len, args.prompt_cap))
               .astype(np.int32) for r in trace}
    mine = trace[rank::world]
    cap_pos = max(len(prompts[r.id]) + r.true_len for r in trace)   # any request may land here
    cap_gen = max(r.true_len for r in trace)
    B = len(mine)
    w = init_weights(s, seed=0, device="cuda")
    m = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=cap_pos + 2 * K + 8, max_tokens=B * (K + 1),
                    max_seqs=B)
    del w
    pr = [prompts[r.id] for r in mine]
    lens = [r.true_len for r in mine]
    plain = RolloutEngine(m, pr, lens, k=0, history=1)
    plain.prefill()
    plain.capture()
    plain.run()
    truth = plain.outputs()
    del plain
    drafter = SyntheticDrafter(truth, mine, scenarios.DEFAULT_METHOD, seed=0, vocab=s.vocab, capacity=cap_gen)
    eng = RolloutEngine(m, pr, lens, k=K, drafters=(drafter,), bonus_token=False, history=1, capacity=cap_pos)
    eng.prefill()
    hook = StragglerPull(dist, {r.id: r for r in trace}, interval=args.interval) if args.pull else None
    drv = RolloutDriver(eng, mine, [scenarios.DEFAULT_METHOD], bon_on_drain=False,
                        priors=scenarios.estimator_priors(), straggler=hook)
    if hook is not None:
        hook.warmup(eng.dev)
    dist.barrier()
    torch.cuda.synchronize()
    rep = drv.run()
    outs = drv.outputs_by_id()
    truth_by_id = {r.id: t for r, t in zip(mine, truth)}
    gathered: list = [None] * world
    dist.all_gather_object(gathered, {"outs": outs, "truth": truth_by_id, "makespan_ms": rep.makespan_ms,
                                      "committed": rep.committed, "steps": rep.steps})
    all_truth, all_outs = {}, {}
    for g in gathered:
        all_truth.update(g["truth"])
        all_outs.update(g["outs"])
    return {"ranks": world, "backend": args.backend, "model": s.name, "batch": args.batch, "pull": bool(args.pull),
            "makespan_ms": round(max(g["makespan_ms"] for g in gathered), 2),
            "rank_makespans_ms": [round(g["makespan_ms"], 2) for g in gathered],
            "committed": int(sum(g["committed"] for g in gathered)),
            "steps": [g["steps"] for g in gathered],
            "moves": len(hook.moves) if hook else 0, "bytes_moved": hook.bytes_moved if hook else 0,
            "exchanges": hook.exchanges if hook else 0,
            "outputs_equal_plain_greedy": all_outs == all_truth}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--batch", type=int, default=512, help="global batch (sharded round-robin)")
    ap.add_argument("--cap", type=int, default=2000, help="true_len cap (reference default 2000)")
    ap.add_argument("--prompt-cap", type=int, default=1 << 30)
    ap.add_argument("--skew", type=int, default=0, help="cut even requests to this length (imbalance)")
    ap.add_argument("--interval", type=int, default=16)
    ap.add_argument("--pull", action="store_true")
    args = ap.parse_args(argv)
    dist.init_process_group(args.backend)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local if args.backend == "nccl" else 0)
    try:
        out = run(args)
        if dist.get_rank() == 0:
            print(json.dumps(out), flush=True)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
