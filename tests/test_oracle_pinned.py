"""CPU: the oracle and the host engine against golden outputs of the reference.

The fixtures were produced by running the unmodified reference package and
vLLM's n-gram proposer (tests/golden/make_golden.py).  These tests pin the
oracle before it is used to judge the CUDA path, and exercise the host-side
round/BoN/reconfig logic with the oracle standing in for the device.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from sim_golden import assert_matches, golden_runs, run_golden

from oracle import ngram_oracle, rollout_oracle


def test_true_tokens_match_reference():
    for rec in golden("keyed_draws.json")["true_sequences"]:
        got = rollout_oracle.true_tokens(rec["seed"], rec["rid"], rec["true_len"])
        assert got.tolist() == rec["tokens"]


def test_accept_uniforms_match_reference():
    for rec in golden("keyed_draws.json")["accept_draws"]:
        got = rollout_oracle._stream(rec["seed"], rec["rid"], "accept_draw",
                                     rec["method"], rec["chunk"]).random(256)
        assert got.tolist() == rec["u"]


def test_config1_golden_hashes():
    # batch 8, n-gram, w=4 -> 860 outcomes, hashes pinned
    runs = {r["name"]: r for r in golden_runs()}
    assert runs["c1-coupled-ngram-w4"]["outcome_key_sha16"] == "4d6f713bb9041822"
    assert runs["c1-decoupled-ngram-w4"]["outcome_key_sha16"] == "65de7cfe6b0c6192"


@pytest.mark.parametrize("rec", golden_runs(), ids=lambda r: f"{r['name']}-b{r['batch']}-s{r['trace_seed']}")
def test_host_engine_with_oracle_reproduces_reference(rec):
    m = run_golden(rec, verifier_factory=rollout_oracle.OracleVerifier)
    assert_matches(rec, m)


def test_ngram_oracle_matches_vllm():
    for case in golden("ngram_vllm.json"):
        got = ngram_oracle.propose(case["ctx"], case["min_n"], case["max_n"], case["k"],
                                   case["max_model_len"])
        assert got == case["draft"], case


def test_verify_window_edge_cases():
    u = np.array([0.1, 0.2, 0.9, 0.1])
    assert rollout_oracle.verify_window(u, 0.5, 0, 4, 3, 10, False) == (2, 3, 1 + 3)
    assert rollout_oracle.verify_window(u, 0.95, 0, 4, 3, 10, False) == (4, 4, 0)
    assert rollout_oracle.verify_window(u, 0.95, 0, 4, 3, 10, True) == (4, 5, 0)
    assert rollout_oracle.verify_window(u, 0.95, 0, 4, 0, 4, True) == (4, 4, 0)  # no bonus at end
    assert rollout_oracle.verify_window(u, 0.05, 0, 4, 0, 10, False) == (0, 1, 3)
    assert rollout_oracle.verify_window(u, 0.5, 3, 0, 0, 10, False) == (0, 1, 0)  # plain


def test_closed_forms_match_reference():
    """Accepted-length law P(a, w) and the expected tokens per window
    (reference costmodel.py:253-284) -- the statistical oracle of §8(a) a14."""
    from paper_2511_16193_b200.costmodel import accept_pmf, expected_tokens_coupled, expected_tokens_decoupled

    rows = golden("closed_forms.json")
    assert len(rows) == 36
    for r in rows:
        p, w = r["p"], r["w"]
        assert [accept_pmf(p, w, a) for a in range(w + 1)] == r["pmf"]
        assert expected_tokens_decoupled(p, w) == r["tau_d"]
        assert expected_tokens_coupled(p, w) == r["tau_c"]
    assert expected_tokens_decoupled(0.5, 3) == 1.0625


def test_gen_trace_matches_reference():
    """Synthetic batch generator (reference workload.py:170-196,
    scenarios.py:71-81): ids, prompt lengths, true lengths and latent
    acceptance rates equal the reference's for two (batch, seed) specs."""
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.workload import gen_trace

    for key, rows in golden("workload.json").items():
        batch, seed = (int(x) for x in key.split("_"))
        tr = gen_trace(scenarios.default_trace_spec(batch=batch, seed=seed))
        assert [[r.id, r.prompt_len, r.true_len, r.latent_accept] for r in tr] == rows
