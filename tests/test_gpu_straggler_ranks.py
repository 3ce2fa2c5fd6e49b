"""Cross-rank straggler pulls on the real engines (reference
``sim.py:546-593`` ``pull_straggler``; ``straggler.StragglerPull`` driving
``migrate.send_requests`` / ``recv_requests``): two prompt-sharded ranks, rank
0's requests cut short so it drains first and adopts rank 1's slowest live
requests mid-rollout -- token rows, KV pages and the reference-acceptance
drafter's rows move, and every request still commits exactly its plain
greedy tokens.

* gloo, both ranks on ONE GPU (host-staged moves; any GPU box)
* NCCL, two GPUs (NVLink P2P; skipped unless two are visible)
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, backend, pull, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT / "scripts"))
    try:
        import straggler_ranks

        argv = ["--backend", backend, "--model", "tiny", "--batch", "16", "--cap", "160", "--prompt-cap", "96",
                "--skew", "6", "--interval", "4"] + (["--pull"] if pull else [])
        import io
        from contextlib import redirect_stdout

        buf = io.StringIO()
        with redirect_stdout(buf):
            straggler_ranks.main(argv)
        q.put(("ok", rank, buf.getvalue()))
    except Exception as e:  # surface worker failures to the test
        q.put(("err", rank, repr(e)))
        raise


def _run(backend, pull):
    import json

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 200 + (0 if backend == "gloo" else 11) + (0 if pull else 23)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, pull, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[0] == "ok", r[2]
    line = next(r[2] for r in res if r[1] == 0)
    return json.loads(line.strip().splitlines()[-1])


@pytest.mark.parametrize("backend", ["gloo", pytest.param("nccl", marks=pytest.mark.skipif(
    torch.cuda.device_count() < 2, reason="needs two GPUs"))])
def test_straggler_pull_moves_requests_and_keeps_outputs(backend):
    out = _run(backend, pull=True)
    assert out["outputs_equal_plain_greedy"]
    assert out["moves"] > 0 and out["bytes_moved"] > 0
    base = _run(backend, pull=False)
    assert base["outputs_equal_plain_greedy"] and base["moves"] == 0
    assert out["committed"] == base["committed"]
