"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (the reference is importable only in the build container):

    python tests/golden/make_golden.py

It imports the unmodified reference package from
/root/reference/pkg/src/specrollout and vLLM 0.22's n-gram proposer, runs
them on seeded inputs, and writes small JSON fixtures.  Nothing at test time
reads /root/reference; the tests read these files.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()[:16]


def outcome_rows(m):
    return [[o.request_id, o.worker, o.method, o.mode, o.window, o.proposed,
             o.accepted, o.committed, o.wasted, int(o.full_accept), o.time_ms]
            for o in m.outcomes]


def request_rows(m):
    return {str(rid): [r.true_len, r.finish_ms, r.committed, r.drafted, r.wasted,
                       r.windows, r.partial_events, r.winner, r.tokens_per_window]
            for rid, r in m.requests.items()}


def gen_sim_runs():
    from specrollout import scenarios
    from specrollout.planner import CoupledPlan, ExecutionPlan
    from specrollout.sim import SimConfig, simulate
    from specrollout.workload import gen_trace

    model = scenarios.default_cost_model()
    bon = list(scenarios.BON_METHODS)
    stacks = {
        "plain": {"policy": "plain"},
        "coupled": {"policy": "coupled"},
        "disaggregated": {"policy": "disaggregated"},
        "decoupled": {"policy": "decoupled"},
        "decoupled+reconfig": {"policy": "decoupled", "reconfig": True},
        "decoupled+bon": {"policy": "decoupled", "bon": True, "bon_methods": bon},
        "decoupled+reconfig+bon": {"policy": "decoupled", "reconfig": True,
                                   "bon": True, "bon_methods": bon},
        "coupled+bonus": {"policy": "coupled", "bonus_token": True},
    }
    runs = []
    for batch, trace_seed in ((10, 0), (10, 1), (12, 5)):
        trace_spec = scenarios.default_trace_spec(batch=batch, seed=trace_seed)
        for name, stack in stacks.items():
            trace = gen_trace(trace_spec)
            kw = dict(stack)
            if "bon_methods" in kw:
                kw["bon_methods"] = tuple(kw["bon_methods"])
            m = simulate(SimConfig(
                trace=trace, model=model, method=scenarios.DEFAULT_METHOD,
                seed=trace_seed, scale_cost=scenarios.default_scale_cost(),
                estimator_priors=scenarios.estimator_priors(), **kw))
            runs.append(_pack(name, batch, trace_seed, trace_seed, stack, m, full=(batch == 10)))
    # config-1-shaped golden: batch 8, n-gram, fixed w=4
    trace = gen_trace(scenarios.default_trace_spec(batch=8, seed=0))
    cp = CoupledPlan(method="ngram", g_v="tp4", window=4, tgs_estimate=1.0,
                     batch_per_group=8, group_gpus=4, g_d=4)
    ep = ExecutionPlan(method="ngram", g_d=1, g_v="tp4", window=4, tgs_estimate=1.0,
                       batch_per_group=8, group_gpus=5)
    for name, kw in (("c1-coupled-ngram-w4", {"policy": "coupled", "coupled_plan": cp}),
                     ("c1-decoupled-ngram-w4", {"policy": "decoupled", "plan": ep})):
        m = simulate(SimConfig(trace=gen_trace(scenarios.default_trace_spec(batch=8, seed=0)),
                               model=model, method="ngram", seed=0,
                               estimator_priors=scenarios.estimator_priors(), **kw))
        stack = {"policy": kw["policy"], "method": "ngram", "window": 4}
        runs.append(_pack(name, 8, 0, 0, stack, m, full=True))
    return runs


def _pack(name, batch, trace_seed, seed, stack, m, full):
    rec = {
        "name": name, "batch": batch, "trace_seed": trace_seed, "seed": seed,
        "stack": stack,
        "makespan_ms": m.makespan_ms, "total_committed": m.total_committed,
        "total_wasted": m.total_wasted, "mean_tgs": m.mean_tgs,
        "bon_assign_count": m.bon_assign_count, "reconfig_count": m.reconfig_count,
        "n_outcomes": len(m.outcomes),
        "outcomes_sha": sha(outcome_rows(m)),
        "sequences_sha": sha({str(k): v for k, v in m.sequences.items()}),
        "events_sha": sha(m.events),
        "requests": request_rows(m),
        "workers": {w: [x.role, x.busy_ms, x.idle_ms, x.drained_ms]
                    for w, x in m.workers.items()},
        "outcome_key_sha16": hashlib.sha256(json.dumps(
            [[o.request_id, o.proposed, o.accepted, o.committed, o.wasted]
             for o in m.outcomes]).encode()).hexdigest()[:16],
    }
    if full:
        rec["outcomes"] = outcome_rows(m)
    if name == "decoupled+reconfig+bon" and trace_seed == 1:
        rec["events"] = m.events  # one full event log for diffing
    return rec


def gen_draws():
    from specrollout.sim import generate_true_sequence
    from specrollout.streams import stream, uniforms

    seqs = []
    for rid, L, seed in ((12, 600, 0), (0, 37, 3), (5, 1000, 1), (3, 256, 2**40 + 9)):
        seqs.append({"rid": rid, "true_len": L, "seed": seed,
                     "tokens": generate_true_sequence(rid, L, seed)})
    draws = []
    for seed, rid, method, chunk in ((0, 0, "draft-0.5b", 0), (1, 7, "ngram", 3),
                                     (2**33 + 1, 2, "draft-1.5b", 1)):
        draws.append({"seed": seed, "rid": rid, "method": method, "chunk": chunk,
                      "u": stream(seed, rid, "accept_draw", method, chunk).random(256).tolist()})
    misc = {"uniforms_5_7_x": uniforms(5, 16, 7, "x").tolist()}
    return {"true_sequences": seqs, "accept_draws": draws, "misc": misc}


def gen_workload():
    from specrollout import scenarios
    from specrollout.workload import gen_trace

    out = {}
    for batch, seed in ((8, 0), (48, 3)):
        tr = gen_trace(scenarios.default_trace_spec(batch=batch, seed=seed))
        out[f"{batch}_{seed}"] = [[r.id, r.prompt_len, r.true_len, r.latent_accept] for r in tr]
    return out


def gen_closed_forms():
    from specrollout.costmodel import accept_pmf, expected_tokens_coupled, expected_tokens_decoupled

    rows = []
    for p in (0.0, 0.1, 0.5, 0.75, 0.9, 1.0):
        for w in (1, 2, 3, 4, 8, 12):
            rows.append({"p": p, "w": w,
                         "pmf": [accept_pmf(p, w, a) for a in range(w + 1)],
                         "tau_d": expected_tokens_decoupled(p, w),
                         "tau_c": expected_tokens_coupled(p, w)})
    return rows


def gen_ngram():
    from vllm.v1.spec_decode.ngram_proposer import _find_longest_matched_ngram_and_propose_tokens as f

    rng = np.random.default_rng(2511)
    cases = []
    for i in range(200):
        length = int(rng.integers(0, 300)) if i % 4 else int(rng.integers(0, 12))
        vocab = int(rng.choice([2, 3, 5, 20, 1000]))
        ctx = rng.integers(0, vocab, size=length).astype(np.int32)
        min_n = int(rng.integers(1, 4))
        max_n = int(rng.integers(min_n, 6))
        k = int(rng.integers(1, 8))
        max_len = int(length + rng.integers(0, 10)) if i % 7 == 0 else 100000
        out = f(ctx, min_n, max_n, max_len, k)
        cases.append({"ctx": ctx.tolist(), "min_n": min_n, "max_n": max_n, "k": k,
                      "max_model_len": max_len, "draft": [int(x) for x in out]})
    return cases


def gen_cli_artifacts():
    """The reference CLI's `simulate` artifacts (cli.py:473-487) for one run,
    as SHA-256 digests of each file's bytes."""
    import tempfile

    from specrollout import cli, scenarios
    from specrollout.sim import SimConfig, simulate
    from specrollout.workload import gen_trace

    bon = tuple(scenarios.BON_METHODS)
    m = simulate(SimConfig(
        trace=gen_trace(scenarios.default_trace_spec(batch=10, seed=1)), model=scenarios.default_cost_model(),
        method=scenarios.DEFAULT_METHOD, seed=1, scale_cost=scenarios.default_scale_cost(),
        estimator_priors=scenarios.estimator_priors(), policy="decoupled", reconfig=True, bon=True,
        bon_methods=bon))
    with tempfile.TemporaryDirectory() as d:
        out = Path(d)
        cli._write_json(out / "summary.json", cli._summary_dict(m))
        cli._write_csv(out / "requests.csv", cli._REQUEST_HEADER, cli._request_rows(m))
        cli._write_csv(out / "workers.csv", cli._WORKER_HEADER, cli._worker_rows(m))
        cli._write_events(out / "events.jsonl", m.events)
        return {"run": {"batch": 10, "trace_seed": 1, "seed": 1, "policy": "decoupled", "reconfig": True,
                        "bon": True},
                "sha256": {f.name: hashlib.sha256(f.read_bytes()).hexdigest() for f in sorted(out.iterdir())}}


def main():
    sys.path.insert(0, str(REF))
    (OUT / "sim_runs.json").write_text(json.dumps(gen_sim_runs()))
    (OUT / "keyed_draws.json").write_text(json.dumps(gen_draws()))
    (OUT / "workload.json").write_text(json.dumps(gen_workload()))
    (OUT / "closed_forms.json").write_text(json.dumps(gen_closed_forms()))
    (OUT / "ngram_vllm.json").write_text(json.dumps(gen_ngram()))
    (OUT / "cli_artifacts.json").write_text(json.dumps(gen_cli_artifacts(), indent=1))
    print("wrote", sorted(p.name for p in OUT.glob("*.json")))


if __name__ == "__main__":
    main()
