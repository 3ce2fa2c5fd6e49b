"""Measured-latency ingestion: time the B200 verify, plain and
draft steps at several batch sizes, fit the reference's affine latency
models (``costmodel.fit_affine``, reference ``costmodel.py:84-102``), write
the cost model in the reference's JSON wire format, and run the reference's
plan search (Alg. 1, ``planner.search_plan`` / ``search_plan_coupled``) on it
for an 8-GPU box.

    python scripts/calibrate_costmodel.py [--model qwen2.5-1.5b] [--out profiles/r01/costmodel_b200.json]

Each latency is one CUDA-graph replay of the step's forward (verify: b
requests x (w + 1) rows over ~600-token contexts; plain: w = 0; draft:
the n-gram kernel per window, or one 0.5B-shaped decode step per token).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2511_16193_b200 import _native  # noqa: E402
from paper_2511_16193_b200.artifacts import write_samples  # noqa: E402
from paper_2511_16193_b200.costmodel import CostModel, ProfileSample, VerifyConfig, fit_affine  # noqa: E402
from paper_2511_16193_b200.model import DeviceModel, init_weights, seq_table, shape  # noqa: E402
from paper_2511_16193_b200.planner import search_plan, search_plan_coupled  # noqa: E402

CTX = 600
BATCHES = (32, 64, 128, 256)


def graph_ms(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin()
        fn()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def model_step_ms(m: DeviceModel, b: int, rows_per: int) -> float:
    dev = m.dev
    M = b * rows_per
    seqs = seq_table([(i * rows_per, rows_per, i, CTX, -1) for i in range(b)], dev)
    tok = torch.randint(0, m.s.vocab, (M,), dtype=torch.int32, device=dev)
    pos = torch.tensor([CTX + j for _ in range(b) for j in range(rows_per)], dtype=torch.int32, device=dev)
    out = torch.empty(M, dtype=torch.int32, device=dev)
    return graph_ms(lambda: m.forward(tok, pos, seqs, num_seqs=b, max_q_len=rows_per,
                                      max_key=CTX + rows_per - 1, out=out))


def ngram_ms(b: int, k: int) -> float:
    lib = _native.lib()
    L = CTX + 64
    tokens = torch.randint(0, 200, (b, L), dtype=torch.int32, device="cuda")
    lens = torch.full((b,), CTX, dtype=torch.int32, device="cuda")
    drafts = torch.empty((b, k), dtype=torch.int32, device="cuda")
    nd = torch.empty(b, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(2 * b, dtype=torch.int64, device="cuda")
    return graph_ms(lambda: _native.check(lib.sr_ngram_propose(
        b, tokens.data_ptr(), L, lens.data_ptr(), 1, 3, k, drafts.data_ptr(), nd.data_ptr(),
        scratch.data_ptr(), _native.stream_handle()), "ngram"))   # the capture stream


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="qwen2.5-1.5b")
    ap.add_argument("--draft-model", default="qwen2.5-0.5b")
    ap.add_argument("--k", type=int, default=4)
    ap.add_argument("--total-gpus", type=int, default=8)
    ap.add_argument("--batch", type=int, default=1024, help="rollout batch for the plan search")
    ap.add_argument("--p", type=float, default=0.7, help="acceptance rate for the plan search")
    ap.add_argument("--out", default=str(Path(__file__).resolve().parent.parent / "profiles" / "r01" /
                                         "costmodel_b200.json"))
    a = ap.parse_args()
    torch.manual_seed(0)
    bmax = max(BATCHES)
    cfg_id = "1xB200"

    def make(name):
        s = shape(name)
        return DeviceModel(s, init_weights(s, seed=0, device="cuda"), dtype="bf16", max_requests=bmax,
                           max_len=CTX + 2 * a.k + 64, max_tokens=bmax * (a.k + 1), max_seqs=bmax)

    samples = {}
    target = make(a.model)
    for w in range(0, a.k + 1):
        key = f"plain/{cfg_id}" if w == 0 else f"verify/{cfg_id}/{w}"
        samples[key] = [ProfileSample(b, model_step_ms(target, b, w + 1), key) for b in BATCHES]
    del target
    torch.cuda.empty_cache()
    samples["draft/ngram/1"] = [ProfileSample(b, ngram_ms(b, a.k) / a.k, "draft/ngram/1") for b in BATCHES]
    drafter = make(a.draft_model)
    samples["draft/draft-0.5b/1"] = [ProfileSample(b, model_step_ms(drafter, b, 1), "draft/draft-0.5b/1")
                                     for b in BATCHES]
    del drafter

    fits = {k: fit_affine(v) for k, v in samples.items()}
    model = CostModel(
        draft={"ngram": {1: fits["draft/ngram/1"]}, "draft-0.5b": {1: fits["draft/draft-0.5b/1"]}},
        verify={cfg_id: {w: fits[f"verify/{cfg_id}/{w}"] for w in range(1, a.k + 1)}},
        plain={cfg_id: fits[f"plain/{cfg_id}"]},
        total_gpus=a.total_gpus,
        configs=[VerifyConfig(id=cfg_id, gpus=1, parallelism="replica")])
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    model.save(a.out)
    # the reference CLI's `fit` input (b,latency_ms,key), next to the model
    write_samples(Path(a.out).with_name("costmodel_samples.csv"), [s for v in samples.values() for s in v])
    report = {"samples_ms": {k: {s.b: round(s.latency_ms, 4) for s in v} for k, v in samples.items()},
              "costmodel": str(Path(a.out).resolve().relative_to(Path(__file__).resolve().parent.parent))
              if Path(a.out).resolve().is_relative_to(Path(__file__).resolve().parent.parent) else a.out,
              "plans": {}}
    for method in ("ngram", "draft-0.5b"):
        d = search_plan(a.batch, model, a.p, method)
        c = search_plan_coupled(a.batch, model, a.p, method)
        report["plans"][method] = {
            "decoupled": {"g_d": d.g_d, "g_v": d.g_v, "window": d.window, "group_gpus": d.group_gpus,
                          "batch_per_group": d.batch_per_group, "tgs_estimate": d.tgs_estimate},
            "coupled": {"g_v": c.g_v, "window": c.window, "group_gpus": c.group_gpus,
                        "batch_per_group": c.batch_per_group, "tgs_estimate": c.tgs_estimate}}
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
