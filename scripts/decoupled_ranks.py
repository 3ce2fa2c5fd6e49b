"""Decoupled speculation across GPUs (configs[3] shape): ranks [0, D) draft,
the rest verify; per round one NCCL P2P exchange per (drafter, verifier).

    torchrun --nproc-per-node 2 scripts/decoupled_ranks.py --drafters 1 --check
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200 import scenarios  # noqa: E402
from paper_2511_16193_b200.decoupled import pairing, run_ranks  # noqa: E402
from paper_2511_16193_b200.dist import shard  # noqa: E402
from paper_2511_16193_b200.engine import ModelDrafter, NgramDrafter, RolloutEngine, SyntheticDrafter  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, shape  # noqa: E402
from paper_2511_16193_b200.streams import stream  # noqa: E402
from paper_2511_16193_b200.workload import gen_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--drafters", type=int, default=1)
    ap.add_argument("--batch", type=int, default=64, help="prompts per verifier")
    ap.add_argument("--model", default="tiny")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--method", default="draft-0.5b")
    ap.add_argument("--drafter", choices=["synthetic", "model", "ngram"], default="synthetic",
                    help="synthetic: reference accept_draw law over the target's greedy continuation; "
                         "model: a random-init --draft-model decoder on the drafter GPU (K5); ngram: K4")
    ap.add_argument("--draft-model", default="qwen2.5-0.5b")
    ap.add_argument("--cap", type=int, default=300, help="max generated tokens per request")
    ap.add_argument("--check", action="store_true", help="compare outputs with plain decoding")
    ap.add_argument("--steady", type=int, default=0,
                    help="steady-state mode: no request finishes; time this many rounds after 5 warm-up "
                         "rounds (the coupled bench's regime) instead of the long-tail trace")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    s = shape(a.model, a.layers)
    nv = world - a.drafters
    trace_all = gen_trace(scenarios.default_trace_spec(batch=a.batch * nv, seed=0))
    shards, traces = {}, {}
    for i, v in enumerate(range(a.drafters, world)):
        tr = shard(trace_all, i, nv)
        prompts = [stream(0, r.id, "prompt").integers(0, s.vocab, size=r.prompt_len).astype(np.int32) for r in tr]
        lens = [min(r.true_len, a.cap) for r in tr]
        if a.steady:
            lens = [(a.steady + 8) * (a.k + 1) + 8] * len(tr)   # budget outlasts the timed rounds
        shards[v] = (prompts, lens)
        traces[v] = tr
    truth = {}
    model = None
    if rank >= a.drafters:
        prompts, lens = shards[rank]
        model = DeviceModel(s, init_weights(s, seed=0, device="cuda"), dtype="bf16", max_requests=len(prompts),
                            max_len=max(len(p) + L for p, L in zip(prompts, lens)) + 2 * a.k + 16,
                            max_tokens=len(prompts) * (a.k + 1), max_seqs=len(prompts))
        plain = RolloutEngine(model, prompts, lens, k=0, history=1)
        plain.prefill()
        plain.run()
        t = plain.outputs()
        width = max(lens)
        mat = torch.full((len(t), width), 0, dtype=torch.int32, device="cuda")
        for b, row in enumerate(t):
            mat[b, : len(row)] = torch.tensor(row, dtype=torch.int32)
        truth[rank] = t
        dist.send(mat, pairing(world, a.drafters)[rank])
    else:
        for v, d in pairing(world, a.drafters).items():
            if d == rank:
                lens = shards[v][1]
                mat = torch.empty((len(lens), max(lens)), dtype=torch.int32, device="cuda")
                dist.recv(mat, v)
                truth[v] = [mat[b, :L].tolist() for b, L in enumerate(lens)]
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    def make_drafter(v):
        if a.drafter == "synthetic":
            return SyntheticDrafter(truth[v], traces[v], a.method, 0, vocab=s.vocab)
        if a.drafter == "ngram":
            return NgramDrafter()
        ds = shape(a.draft_model)
        prompts, lens = shards[v]
        B = len(prompts)
        max_len = max(len(p) + L for p, L in zip(prompts, lens)) + 4 * a.k + 32
        dm = DeviceModel(ds, init_weights(ds, seed=1, device="cuda"), dtype="bf16", max_requests=B,
                         max_len=max_len, max_tokens=B * (a.k + 2), max_seqs=B)
        return ModelDrafter(dm)

    times = []
    outs, rows, rounds = run_ranks(
        dist, rank, world, a.drafters, shards, a.k,
        make_drafter=make_drafter,
        make_model=lambda: model, max_rounds=(a.steady + 6) if a.steady else 1_000_000, round_times=times)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res = {"rank": rank, "rounds": rounds, "seconds": dt}
    if rank >= a.drafters:
        committed = int(sum(len(o) for o in outs))
        res.update(committed=committed, tokens_per_s=committed / dt,
                   mean_accepted=float(rows[:, :, 1][rows[:, :, 0] > 0].mean()))
        if a.steady:
            verify_ms = times.pop()   # per-round device time of the verify graph
            # rows[i] = outcome of round i + 1; timed rounds 6 .. steady + 5
            w0 = 5
            res["steady_verify_ms_per_round"] = float(np.mean(verify_ms[w0:w0 + a.steady]))
            dt_s = times[w0 + a.steady - 1] - times[w0 - 1]
            c = int(rows[w0 - 1:w0 - 1 + a.steady, :, 2].clip(min=0).sum())
            res.update(steady_rounds=a.steady, steady_committed=c, steady_tokens_per_s=c / dt_s,
                       steady_ms_per_round=dt_s * 1e3 / a.steady)
        if a.check:
            res["outputs_equal_plain"] = (all(o == t[: len(o)] for o, t in zip(outs, truth[rank])) if a.steady
                                          else outs == truth[rank])
    print(json.dumps(res), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
