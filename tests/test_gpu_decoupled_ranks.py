"""Decoupled speculation across processes (configs[3] placement, reference
``sim.py:860-917`` / ``1051-1092``): a drafter rank and a verifier rank run
``decoupled.run_ranks`` and exchange windows and decisions every round.

* ``HostChannel`` over gloo with both ranks on ONE GPU (runs on any GPU box):
  the cross-process protocol reproduces the reference simulator's decoupled
  golden outcome stream (``c1-decoupled-ngram-w4``), depth-2 waste included.
* ``NcclChannel`` over NVLink with the ranks on two GPUs (skipped unless two
  are visible): the same golden.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _setup():
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.engine import RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape
    from paper_2511_16193_b200.streams import stream
    from paper_2511_16193_b200.workload import gen_trace

    trace = gen_trace(scenarios.default_trace_spec(batch=8, seed=0))
    s = shape("tiny")
    prompts = [stream(0, r.id, "prompt").integers(0, s.vocab, size=r.prompt_len).astype(np.int32) for r in trace]
    lens = [r.true_len for r in trace]
    max_len = max(len(p) + L for p, L in zip(prompts, lens)) + 16

    def model():
        return DeviceModel(s, init_weights(s, seed=0), dtype="bf16", max_requests=8, max_len=max_len,
                           max_tokens=2048, max_seqs=24)

    m = model()
    plain = RolloutEngine(m, prompts, lens, k=0, history=1)
    plain.prefill()
    plain.run()
    return s, trace, prompts, lens, m, plain.outputs()


def _worker(rank, world, port, backend, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist

    from paper_2511_16193_b200.decoupled import HostChannel, NcclChannel, run_ranks
    from paper_2511_16193_b200.engine import SyntheticDrafter

    torch.cuda.set_device(rank if backend == "nccl" else 0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        s, trace, prompts, lens, m, truth = _setup()
        shards = {1: (prompts, lens)}
        outs, rows, rounds = run_ranks(
            dist, rank, world, 1, shards, 4,
            make_drafter=lambda v: SyntheticDrafter(truth, trace, "ngram", 0, vocab=s.vocab),
            make_model=lambda: m, channel=HostChannel if backend == "gloo" else NcclChannel)
        if rank == 1:
            q.put(("ok", outs == truth, rows.tolist(), [r.id for r in trace], rounds))
        else:
            q.put(("ok", None, None, None, rounds))
    except Exception as e:  # surface worker failures to the test
        q.put(("err", repr(e), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def _run(backend):
    from conftest import golden

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + os.getpid() % 200 + (0 if backend == "gloo" else 7)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[0] == "ok", r[1]
    ver = next(r for r in res if r[1] is not None)
    _, same, rows, rids, rounds = ver
    assert same, "decoupled output differs from plain greedy"
    rows = np.asarray(rows)
    rec = next(r for r in golden("sim_runs.json") if r["name"] == "c1-decoupled-ngram-w4")
    for b, rid in enumerate(rids):
        got = [tuple(int(x) for x in row) for row in rows[:, b, :] if row[0] or row[2]]
        exp = [tuple(o[5:9]) for o in rec["outcomes"] if o[0] == rid]
        assert got == exp, f"request {rid}"
    drafter_rounds = next(r[4] for r in res if r[1] is None)
    assert drafter_rounds == rounds       # both ranks agree when the rollout ended


def test_decoupled_two_processes_one_gpu_host_channel():
    _run("gloo")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (NVLink P2P)")
def test_decoupled_two_gpus_nccl():
    _run("nccl")
