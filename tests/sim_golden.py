"""Replays the reference golden simulations (tests/golden/sim_runs.json) on
our engine with a given verifier and compares every recorded field."""

from __future__ import annotations

import hashlib
import json

from conftest import golden, make_trace


def sha(obj) -> str:
    return hashlib.sha256(json.dumps(obj, sort_keys=True).encode()).hexdigest()[:16]


def outcome_rows(m):
    return [[o.request_id, o.worker, o.method, o.mode, o.window, o.proposed,
             o.accepted, o.committed, o.wasted, int(o.full_accept), o.time_ms]
            for o in m.outcomes]


def run_golden(rec, verifier_factory=None):
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.planner import CoupledPlan, ExecutionPlan
    from paper_2511_16193_b200.sim import SimConfig, simulate

    model = scenarios.default_cost_model()
    trace = make_trace(rec["batch"], rec["trace_seed"])
    stack = dict(rec["stack"])
    if rec["name"].startswith("c1-"):
        if stack["policy"] == "coupled":
            kw = {"policy": "coupled", "coupled_plan": CoupledPlan(
                method="ngram", g_v="tp4", window=4, tgs_estimate=1.0,
                batch_per_group=8, group_gpus=4, g_d=4)}
        else:
            kw = {"policy": "decoupled", "plan": ExecutionPlan(
                method="ngram", g_d=1, g_v="tp4", window=4, tgs_estimate=1.0,
                batch_per_group=8, group_gpus=5)}
        cfg = SimConfig(trace=trace, model=model, method="ngram", seed=rec["seed"],
                        estimator_priors=scenarios.estimator_priors(), **kw)
    else:
        if "bon_methods" in stack:
            stack["bon_methods"] = tuple(stack["bon_methods"])
        cfg = SimConfig(trace=trace, model=model, method=scenarios.DEFAULT_METHOD,
                        seed=rec["seed"], scale_cost=scenarios.default_scale_cost(),
                        estimator_priors=scenarios.estimator_priors(), **stack)
    return simulate(cfg, verifier_factory=verifier_factory)


def assert_matches(rec, m):
    name = rec["name"]
    if "outcomes" in rec:
        got = outcome_rows(m)
        for i, (g, e) in enumerate(zip(got, rec["outcomes"])):
            assert g == e, f"{name}: outcome {i} differs: {g} != {e}"
        assert len(got) == len(rec["outcomes"]), name
    assert sha(outcome_rows(m)) == rec["outcomes_sha"], name
    assert len(m.outcomes) == rec["n_outcomes"], name
    if "events" in rec:
        for i, (g, e) in enumerate(zip(m.events, rec["events"])):
            assert g == e, f"{name}: event {i} differs: {g} != {e}"
    assert sha(m.events) == rec["events_sha"], name
    assert sha({str(k): v for k, v in m.sequences.items()}) == rec["sequences_sha"], name
    assert m.makespan_ms == rec["makespan_ms"], name
    assert m.total_wasted == rec["total_wasted"], name
    assert m.total_committed == rec["total_committed"], name
    assert m.bon_assign_count == rec["bon_assign_count"], name
    assert m.reconfig_count == rec["reconfig_count"], name
    req = {str(rid): [r.true_len, r.finish_ms, r.committed, r.drafted, r.wasted,
                      r.windows, r.partial_events, r.winner, r.tokens_per_window]
           for rid, r in m.requests.items()}
    assert req == rec["requests"], name
    workers = {w: [x.role, x.busy_ms, x.idle_ms, x.drained_ms] for w, x in m.workers.items()}
    assert workers == rec["workers"], name


def golden_runs():
    return golden("sim_runs.json")
