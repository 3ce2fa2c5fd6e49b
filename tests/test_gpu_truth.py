"""GPU parity: keyed draws, window verification and whole rollouts vs the
reference (golden fixtures) and the CPU oracle."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, make_trace, run_sim
from sim_golden import assert_matches, golden_runs, run_golden

from oracle import rollout_oracle

pytestmark = pytest.mark.gpu


def test_keyed_tokens_bit_exact():
    from paper_2511_16193_b200.sim import generate_true_sequence

    for rec in golden("keyed_draws.json")["true_sequences"]:
        assert generate_true_sequence(rec["rid"], rec["true_len"], rec["seed"]) == rec["tokens"]


def test_keyed_uniforms_bit_exact():
    from paper_2511_16193_b200.verify import entropy_words, keyed_fill

    recs = golden("keyed_draws.json")["accept_draws"]
    streams = [entropy_words(r["seed"], r["rid"], "accept_draw", r["method"], r["chunk"])
               for r in recs]
    out = torch.empty((len(recs), 256), dtype=torch.float64, device="cuda")
    keyed_fill("uniforms", streams, 256, out)
    got = out.cpu().numpy()
    for i, r in enumerate(recs):
        assert got[i].tolist() == r["u"]


def test_keyed_tokens_many_streams_vs_oracle():
    from paper_2511_16193_b200.verify import truth_table

    ids = list(range(0, 300, 7))
    lens = [1 + (i * 37) % 900 for i in range(len(ids))]
    table = truth_table(11, ids, lens).cpu().numpy()
    for i, (rid, L) in enumerate(zip(ids, lens)):
        assert table[i, :L].tolist() == rollout_oracle.true_tokens(11, rid, L).tolist()


def test_verify_windows_random_vs_oracle():
    from paper_2511_16193_b200.verify import DeviceVerifier
    from paper_2511_16193_b200.workload import Request

    rng = np.random.default_rng(0)
    reqs = [Request(id=i, prompt_len=10, true_len=int(rng.integers(1, 700)),
                    latent_accept={"a": float(rng.uniform()), "b": float(rng.uniform())})
            for i in range(64)]
    for bonus in (False, True):
        dev = DeviceVerifier(3, reqs, ["a", "b"], bonus)
        ora = rollout_oracle.OracleVerifier(3, reqs, ["a", "b"], bonus)
        pos = [0] * len(reqs)
        for _ in range(200):
            live = [i for i in range(len(reqs)) if pos[i] < reqs[i].true_len]
            if not live:
                break
            rows = rng.permutation(live)[: int(rng.integers(1, len(live) + 1))]
            method = int(rng.integers(0, 2))
            starts = np.array([pos[r] for r in rows], np.int32)
            ns = np.array([min(int(rng.integers(0, 40)), reqs[r].true_len - pos[r])
                           for r in rows], np.int32)
            extra = rng.integers(0, 5, size=len(rows)).astype(np.int32)
            got = dev.verify(rows.astype(np.int32), method, starts, ns, extra)
            exp = ora.verify(rows, method, starts, ns, extra)
            for g, e in zip(got, exp):
                assert np.array_equal(g, e)
            for r, c in zip(rows, got[1]):
                pos[r] += int(c)
        seqs = dev.sequences()
        for i, r in enumerate(reqs):
            assert seqs[i][: r.true_len] == ora.sequences()[i]


def test_conflicting_commit_detected():
    from paper_2511_16193_b200.verify import DeviceVerifier
    from paper_2511_16193_b200.workload import Request

    reqs = [Request(id=0, prompt_len=1, true_len=50, latent_accept={"m": 0.5})]
    dev = DeviceVerifier(0, reqs, ["m"], False)
    dev.seq[0, 3] = (dev.truth[0, 3] + 1) % 50257   # corrupt a slot
    out = dev.verify(np.array([0], np.int32), 0, np.array([0], np.int32),
                     np.array([10], np.int32), np.array([0], np.int32))
    if out[1][0] > 3:
        assert out[3][0] == -1


@pytest.mark.parametrize("rec", golden_runs(), ids=lambda r: f"{r['name']}-b{r['batch']}-s{r['trace_seed']}")
def test_device_rollout_reproduces_reference(rec):
    assert_matches(rec, run_golden(rec))


STACKS = [
    {"policy": "plain"},
    {"policy": "coupled"},
    {"policy": "disaggregated"},
    {"policy": "decoupled"},
    {"policy": "decoupled", "reconfig": True},
    {"policy": "decoupled", "bon": True, "bon_methods": ("ngram", "draft-1.5b")},
    {"policy": "decoupled", "reconfig": True, "bon": True,
     "bon_methods": ("ngram", "draft-1.5b")},
]


@pytest.mark.parametrize("stack", STACKS)
def test_sequences_identical_to_truth(model, stack):
    # reference tests/test_sim.py:25-33 on the device engine
    from paper_2511_16193_b200.sim import generate_true_sequence

    for seed in (0, 1):
        trace = make_trace(batch=10, seed=seed)
        m = run_sim(model, trace, seed, **stack)
        for r in trace:
            assert m.sequences[r.id] == generate_true_sequence(r.id, r.true_len, seed)


@pytest.mark.parametrize("stack", STACKS[1:])
def test_waste_bounds(model, stack):
    # reference tests/test_sim.py:36-44
    m = run_sim(model, make_trace(batch=10, seed=3), 3, **stack)
    assert m.outcomes
    for o in m.outcomes:
        limit = 2 * o.window - 1 if o.mode == "D" else o.window - 1
        assert o.wasted <= limit, o


@pytest.mark.parametrize("p", [0.1, 0.5, 0.9])
def test_synthetic_acceptance_law_matches_pmf(p):
    """The device drafter under the reference's keyed accept_draw law
    (sim.py:322-336): accepted-prefix histogram over 4096 requests x 8 window
    offsets vs the closed form P(a, w) (costmodel.py:253-260), 5-sigma MC
    tolerance, and tau within 2 % (reference tests/test_acceptance.py:85-104)."""
    from paper_2511_16193_b200 import _native
    from paper_2511_16193_b200.costmodel import accept_pmf, expected_tokens_decoupled
    from paper_2511_16193_b200.verify import CHUNK, entropy_words, keyed_fill

    lib = _native.lib()
    R, offsets = 4096, 8
    dev = "cuda"
    uni = torch.empty((R, CHUNK), dtype=torch.float64, device=dev)
    keyed_fill("uniforms", [entropy_words(0, rid, "accept_draw", "draft-0.5b", 0) for rid in range(R)],
               CHUNK, uni)
    truth = torch.zeros((R, CHUNK), dtype=torch.int32, device=dev)
    truth_len = torch.full((R,), CHUNK, dtype=torch.int32, device=dev)
    pr = torch.full((R,), p, dtype=torch.float64, device=dev)
    st = _native.stream_handle()
    for w in (1, 2, 4, 8):
        counts = np.zeros(w + 1, dtype=np.int64)
        for off in range(offsets):
            gen = torch.full((R,), off * 16, dtype=torch.int32, device=dev)
            drafts = torch.full((R, w), -1, dtype=torch.int32, device=dev)
            nd = torch.zeros(R, dtype=torch.int32, device=dev)
            _native.check(lib.sr_synthetic_draft(R, w, truth.data_ptr(), CHUNK, truth_len.data_ptr(),
                                                 uni.data_ptr(), CHUNK, pr.data_ptr(), gen.data_ptr(), 50257,
                                                 drafts.data_ptr(), nd.data_ptr(), st), "sr_synthetic_draft")
            d = drafts.cpu().numpy()
            assert (nd.cpu().numpy() == w).all()
            hit = d == 0                       # proposed the true token
            a = np.where(hit.all(1), w, (~hit).argmax(1))
            counts += np.bincount(a, minlength=w + 1)
        n = counts.sum()
        freq = counts / n
        pmf = np.array([accept_pmf(p, w, a) for a in range(w + 1)])
        sigma = np.sqrt(pmf * (1 - pmf) / n)
        assert np.all(np.abs(freq - pmf) <= 5 * sigma + 1e-9), (w, freq, pmf)
        a_vals = np.arange(w + 1)
        tau = float((freq * np.where(a_vals < w, (a_vals + 1) / 2.0, float(w))).sum())
        assert abs(tau - expected_tokens_decoupled(p, w)) / expected_tokens_decoupled(p, w) < 0.02
