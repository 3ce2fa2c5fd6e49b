"""K3 rejection-sampling mode (Leviathan speculative sampling; semantics of
vLLM 0.22 rejection_sampler.py:708-760) for stochastic drafters.

* Kernel level (``sr_accept_rejection`` through the C-ABI): over 60K
  independent requests with the same target p and drafter q, the first
  committed token follows p (chi-square), the bonus after a full accept
  follows p_1, and drafts are accepted at rate sum_v min(p_v, q_v).
* Engine level: a drafter that IS the target (q == p bit for bit: the verify
  and decode logits are batch invariant) has every draft accepted; a
  perturbed drafter is accepted at least as often as under the Gumbel-coupled
  exact-match mode (which no coupling can beat Leviathan's optimum).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch
from scipy import stats as sstats

pytestmark = pytest.mark.gpu


def _softmax(x):
    e = np.exp(x - x.max())
    return e / e.sum()


def test_rejection_kernel_preserves_target_distribution():
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    rng = np.random.default_rng(0)
    V, B, ctx = 8, 60000, 10
    lp0 = rng.normal(0, 1.2, V).astype(np.float32)
    lp1 = rng.normal(0, 1.2, V).astype(np.float32)
    lq = (lp0 + rng.normal(0, 1.0, V)).astype(np.float32)
    p0, p1, q = _softmax(lp0.astype(np.float64)), _softmax(lp1.astype(np.float64)), _softmax(lq.astype(np.float64))
    d = rng.choice(V, size=B, p=q).astype(np.int32)          # the drafter's samples from q
    seqs = np.zeros((B, 8), np.int32)
    seqs[:, 0] = np.arange(B) * 2
    seqs[:, 1] = 2
    seqs[:, 2] = np.arange(B)
    seqs[:, 3] = ctx
    seqs[:, 4] = -1
    token_ids = np.zeros(2 * B, np.int32)
    token_ids[1::2] = d
    p_logits = np.stack([lp0, lp1] * B).astype(np.float32)    # row 2b: slot 0, row 2b+1: bonus slot
    q_logits = np.tile(lq, (1, B, 1)).astype(np.float32)
    stride = 32
    dev = {k: torch.from_numpy(v).cuda() for k, v in dict(
        seqs=seqs, token_ids=token_ids, p=p_logits, q=q_logits,
        tokens=np.zeros((B, stride), np.int32), seq_len=np.full(B, ctx + 1, np.int32),
        gen_len=np.zeros(B, np.int32), max_new=np.full(B, 8, np.int32)).items()}
    stats_ws = torch.zeros(int(lib.sr_accept_rejection_workspace_floats(B, 1)), dtype=torch.float32, device="cuda")
    outcome = torch.zeros((B, 4), dtype=torch.int32, device="cuda")
    bon = torch.zeros(B, dtype=torch.int32, device="cuda")
    _native.check(lib.sr_accept_rejection(
        B, 1, dev["seqs"].data_ptr(), dev["token_ids"].data_ptr(), dev["p"].data_ptr(), V, dev["q"].data_ptr(), V,
        V, 1.0, 1234, dev["tokens"].data_ptr(), stride, dev["seq_len"].data_ptr(), dev["gen_len"].data_ptr(),
        dev["max_new"].data_ptr(), 1, stats_ws.data_ptr(), outcome.data_ptr(), bon.data_ptr(),
        _native.stream_handle()), "sr_accept_rejection")
    torch.cuda.synchronize()
    out = outcome.cpu().numpy()
    toks = dev["tokens"].cpu().numpy()
    acc = out[:, 1] == 1
    # outcome rows: (proposed 1, accepted a, committed a + 1 (bonus on), wasted)
    assert (out[:, 0] == 1).all()
    assert (out[:, 2] == out[:, 1] + 1).all()
    assert (out[:, 3] == np.where(acc, 0, 0)).all()
    # acceptance rate == sum min(p, q)
    rate, exp_rate = acc.mean(), np.minimum(p0, q).sum()
    assert abs(rate - exp_rate) < 5 * np.sqrt(exp_rate * (1 - exp_rate) / B), (rate, exp_rate)
    # accepted slots keep the draft; the first committed token follows p0
    assert (toks[acc, ctx + 1] == d[acc]).all()
    first = np.bincount(toks[:, ctx + 1], minlength=V)
    assert sstats.chisquare(first, p0 * B).pvalue > 1e-4, (first, p0 * B)
    # after a full accept the bonus is the target's sample of p1
    second = np.bincount(toks[acc, ctx + 2], minlength=V)
    assert sstats.chisquare(second, p1 * acc.sum()).pvalue > 1e-4, (second, p1 * acc.sum())
    assert (dev["gen_len"].cpu().numpy() == out[:, 2]).all()


def _perturbed(w, scale, seed):
    g = torch.Generator().manual_seed(seed)

    def p(t):
        return t + torch.randn(t.shape, generator=g) * 0.02 * scale

    emb = p(w["embed"])
    return {"embed": emb, "lm_head": emb, "final_norm": w["final_norm"],
            "layers": [{k: p(v) for k, v in L.items()} for L in w["layers"]]}


def test_rejection_mode_engine_acceptance():
    from paper_2511_16193_b200.engine import ModelDrafter, RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    B, k, T = 8, 4, 1.0
    s = shape("tiny")
    w = init_weights(s, seed=0)
    m = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=256, max_tokens=512, max_seqs=B,
                    logits_capacity=B * (k + 1))
    rng = np.random.default_rng(4)
    prompts = [rng.integers(0, s.vocab, int(rng.integers(20, 60))).astype(np.int32) for _ in range(B)]
    max_new = [48] * B

    def drafter(wd):
        return ModelDrafter(DeviceModel(s, wd, dtype="bf16", max_requests=B, max_len=256, max_tokens=512,
                                        max_seqs=B, logits_capacity=B))

    def run(wd, acceptance):
        eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(drafter(wd),), history=256, temperature=T,
                            seed=17, acceptance=acceptance)
        eng.prefill()
        steps = eng.run()
        rows = eng.outcome_rows(steps).reshape(-1, 4)
        live = rows[rows[:, 0] > 0]
        assert [len(o) for o in eng.outputs()] == max_new
        return live[:, 1].sum(), live[:, 0].sum()

    a, n = run(w, "rejection")
    assert a == n                       # q == p: every draft accepted
    wd = _perturbed(w, 0.6, 1)
    a_rs, n_rs = run(wd, "rejection")
    a_gc, n_gc = run(wd, "exact")       # Gumbel-coupled exact match, same drafter
    r_rs, r_gc = a_rs / n_rs, a_gc / n_gc
    sd = np.sqrt(r_rs * (1 - r_rs) / n_rs + r_gc * (1 - r_gc) / n_gc)
    assert r_rs >= r_gc - 3 * sd, (r_rs, r_gc)


def test_rejection_mode_config_errors():
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine
    from paper_2511_16193_b200.errors import ConfigError
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    s = shape("tiny")
    m = DeviceModel(s, init_weights(s, seed=0), dtype="bf16", max_requests=2, max_len=128, max_tokens=64,
                    max_seqs=2, logits_capacity=10)
    p = [np.arange(5, dtype=np.int32)] * 2
    with pytest.raises(ConfigError):
        RolloutEngine(m, p, [4, 4], k=4, drafters=(NgramDrafter(),), temperature=1.0, acceptance="rejection")
    with pytest.raises(ConfigError):
        RolloutEngine(m, p, [4, 4], k=4, acceptance="leviathan")
