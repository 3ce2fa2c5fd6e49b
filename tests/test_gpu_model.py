"""GPU parity of the model-mode rollout: verify-forward logits vs the CPU
oracle (1e-5 fp32, 1e-2 bf16, as BASELINE.json's north star states), greedy
outputs vs the oracle, and the exactness invariant: plain decode, n-gram
speculation and Best-of-N commit byte-identical sequences."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ngram_oracle
from oracle.qwen2_oracle import Qwen2Oracle, margin

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
BF16_TOL = 1e-2


def rel_err(got: torch.Tensor, exp: torch.Tensor) -> float:
    return float((got.double() - exp.double()).abs().max() / exp.double().abs().max())


def prompts_for(vocab: int, n: int, seed: int, lo=20, hi=90, alphabet=40):
    rng = np.random.default_rng(seed)
    words = rng.integers(0, vocab, size=alphabet)
    return [words[rng.integers(0, alphabet, size=int(rng.integers(lo, hi)))].astype(np.int32)
            for _ in range(n)]


def make(shape_name, dtype, layers=None, B=4, max_len=512, branches=0, logits=0, max_tokens=None):
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    s = shape(shape_name, layers)
    w = init_weights(s, seed=0)
    m = DeviceModel(s, w, dtype=dtype, max_requests=B, max_len=max_len,
                    max_tokens=max_tokens or max(B * 8 * 3, 512), max_seqs=B * 3,
                    branches=branches, logits_capacity=logits)
    return s, w, m


def prefill_logits(m, prompts):
    """Logits of every prompt position through the GPU prefill path."""
    from paper_2511_16193_b200.model import seq_table

    rows, ids, pos, start = [], [], [], 0
    for b, p in enumerate(prompts):
        rows.append((start, len(p), b, 0, -1))
        ids.append(torch.from_numpy(p))
        pos.append(torch.arange(len(p), dtype=torch.int32))
        start += len(p)
    ids = torch.cat(ids).cuda()
    pos = torch.cat(pos).cuda()
    out = torch.empty(start, m.s.vocab, device="cuda")
    m.forward(ids, pos, seq_table(rows, "cuda"), num_seqs=len(rows),
              max_q_len=max(len(p) for p in prompts), max_key=max(len(p) for p in prompts) - 1,
              out=out, output=1)
    torch.cuda.synchronize()
    res, start = [], 0
    for p in prompts:
        res.append(out[start:start + len(p)].cpu())
        start += len(p)
    return res


@pytest.mark.parametrize("dtype,tol", [("fp32", FP32_TOL), ("bf16", BF16_TOL)])
def test_tiny_prefill_logits_vs_oracle(dtype, tol):
    s, w, m = make("tiny", dtype, logits=4096)
    ora = Qwen2Oracle(s, w, dtype)
    prompts = prompts_for(s.vocab, 3, 1)
    for p, got in zip(prompts, prefill_logits(m, prompts)):
        assert rel_err(got, ora.logits(p.tolist())) <= tol


def test_qwen15b_shape_bf16_logits_vs_oracle():
    # real Qwen2.5-1.5B widths (hidden 1536, 12/2 heads, hd 128, vocab 151936), 2 layers
    s, w, m = make("qwen2.5-1.5b", "bf16", layers=2, B=2, logits=512)
    ora = Qwen2Oracle(s, w, "bf16")
    prompts = prompts_for(s.vocab, 2, 2, lo=70, hi=140)
    for p, got in zip(prompts, prefill_logits(m, prompts)):
        assert rel_err(got, ora.logits(p.tolist())) <= BF16_TOL


def run_engine(m, prompts, max_new, k, drafters=None, bonus=False):
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    eng = RolloutEngine(m, prompts, max_new, k=k, drafters=drafters or (NgramDrafter(),),
                        bonus_token=bonus, history=512)
    eng.prefill()
    steps = eng.run()
    return eng, steps


@pytest.mark.parametrize("bonus", [False, True])
def test_tiny_fp32_spec_decode_matches_oracle(bonus):
    s, w, m = make("tiny", "fp32", logits=64)
    ora = Qwen2Oracle(s, w, "fp32")
    prompts = prompts_for(s.vocab, 4, 3)
    max_new = [40, 17, 33, 5]
    eng, steps = run_engine(m, prompts, max_new, k=4, bonus=bonus)
    outs = eng.outputs()
    rows = eng.outcome_rows(steps)
    for b, p in enumerate(prompts):
        exp, exp_rows = ora.spec_decode(p.tolist(), max_new[b], 4, bonus=bonus,
                                        max_model_len=eng.stride)
        assert outs[b] == exp, f"request {b}"
        got_rows = [tuple(r) for r in rows[:, b, :] if r[0] or r[2]]
        assert got_rows == exp_rows, f"request {b} outcomes"


def test_tiny_fp32_greedy_margins():
    # parity above is only meaningful if greedy choices are not near-ties
    s, w, _ = make("tiny", "fp32")
    ora = Qwen2Oracle(s, w, "fp32")
    p = prompts_for(s.vocab, 1, 3)[0].tolist()
    lg = ora.logits(p + ora.greedy(p, 8))
    assert min(margin(r) for r in lg[len(p) - 1:]) > 1e-4


@pytest.mark.parametrize("shape_name,layers", [("tiny", None), ("qwen2.5-1.5b", 2)])
def test_bf16_spec_equals_plain_bit_exact(shape_name, layers):
    """Exactness invariant: plain decode, k=4 n-gram speculation
    and Best-of-N (3 n-gram drafters) commit identical sequences."""
    from paper_2511_16193_b200.engine import NgramDrafter

    B = 4
    s, w, m = make(shape_name, "bf16", layers=layers, B=B, branches=2 * B, max_len=512)
    prompts = prompts_for(s.vocab, B, 4)
    max_new = [60, 31, 47, 12]
    plain, _ = run_engine(m, prompts, max_new, k=0)
    ref = plain.outputs()
    spec, _ = run_engine(m, prompts, max_new, k=4)
    assert spec.outputs() == ref
    bon, _ = run_engine(m, prompts, max_new, k=4,
                        drafters=(NgramDrafter(1, 3), NgramDrafter(2, 4), NgramDrafter(1, 1)))
    assert bon.outputs() == ref


def test_verify_logits_equal_decode_logits_bit_exact():
    """A position's logits are bit-identical in a 5-row verify window and in
    a 1-row decode step (batch-invariant GEMM + absolute-position attention)."""
    from paper_2511_16193_b200.model import seq_table

    s, w, m = make("tiny", "bf16", B=1, logits=256)
    p = prompts_for(s.vocab, 1, 5)[0]
    L = len(p)
    ids = torch.from_numpy(p).cuda()
    pos = torch.arange(L, dtype=torch.int32, device="cuda")
    full = torch.empty(L, s.vocab, device="cuda")
    # prefill the first L-5 tokens, then verify the last 5 as one window
    P = L - 5
    m.forward(ids[:P], pos[:P], seq_table([(0, P, 0, 0, -1)], "cuda"), num_seqs=1, max_q_len=P,
              max_key=P - 1, out=full[:P], output=1)
    win = torch.empty(5, s.vocab, device="cuda")
    m.forward(ids[P:], pos[P:], seq_table([(0, 5, 0, P, -1)], "cuda"), num_seqs=1, max_q_len=5,
              max_key=L - 1, out=win, output=1)
    # now decode the same 5 positions one at a time (KV rewritten in place)
    for j in range(5):
        one = torch.empty(1, s.vocab, device="cuda")
        m.forward(ids[P + j:P + j + 1], pos[P + j:P + j + 1], seq_table([(0, 1, 0, P + j, -1)], "cuda"),
                  num_seqs=1, max_q_len=1, max_key=P + j, out=one, output=1)
        torch.cuda.synchronize()
        assert torch.equal(one[0], win[j]), f"slot {j}"


@pytest.mark.parametrize("shape_name,layers", [("tiny", None), ("qwen2.5-1.5b", 2)])
def test_small_m_window_logits_equal_large_prefill_bit_exact(shape_name, layers):
    """Positions prefilled in one 300-row forward (large-M GEMM mode) and
    re-verified as a 6-row window (small-M mode: weights as the UMMA M side,
    K ranges summed in order, fused qkv-RoPE / residual-RMSNorm epilogues
    through the transpose) give bit-identical logits."""
    from paper_2511_16193_b200 import _native
    from paper_2511_16193_b200.model import seq_table

    lib = _native.lib()
    _native.check(lib.sr_set_gemm_swap_max_m(128), "swap threshold")  # every projection, any size
    try:
        s, w, m = make(shape_name, "bf16", layers=layers, B=1, logits=512, max_len=512)
    finally:
        _native.check(lib.sr_set_gemm_swap_max_m(-1), "swap threshold")
    rng = np.random.default_rng(3)
    L = 300
    ids = torch.from_numpy(rng.integers(0, s.vocab, L).astype(np.int32)).cuda()
    pos = torch.arange(L, dtype=torch.int32, device="cuda")
    full = torch.empty(L, s.vocab, device="cuda")
    m.forward(ids, pos, seq_table([(0, L, 0, 0, -1)], "cuda"), num_seqs=1, max_q_len=L, max_key=L - 1,
              out=full, output=1)
    P = L - 6
    win = torch.empty(6, s.vocab, device="cuda")
    m.forward(ids[P:], pos[P:], seq_table([(0, 6, 0, P, -1)], "cuda"), num_seqs=1, max_q_len=6,
              max_key=L - 1, out=win, output=1)
    torch.cuda.synchronize()
    assert torch.equal(win, full[P:])


def test_accept_commit_kernel_vs_python():
    """K3 on random verify batches (N=3 drafters, budgets, bonus) vs a direct
    restatement of sim.py:983-1042 + longest-prefix Best-of-N."""
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    rng = np.random.default_rng(7)
    B, N, k = 37, 3, 5
    for bonus in (0, 1):
        S = B * N
        seqs = np.zeros((S, 8), np.int32)
        token_ids = rng.integers(0, 4, size=S * (k + 1)).astype(np.int32)
        target = rng.integers(0, 4, size=S * (k + 1)).astype(np.int32)
        stride = 64
        tokens = np.zeros((B, stride), np.int32)
        seq_len = rng.integers(5, 20, size=B).astype(np.int32)
        gen_len = rng.integers(0, 10, size=B).astype(np.int32)
        max_new = gen_len + rng.integers(0, 8, size=B).astype(np.int32)
        for s_ in range(S):
            seqs[s_, :5] = (s_ * (k + 1), int(rng.integers(0, k + 2)), s_ // N, 0, -1)
        dev = {n: torch.from_numpy(v).cuda() for n, v in dict(
            seqs=seqs, token_ids=token_ids, target=target, tokens=tokens, seq_len=seq_len,
            gen_len=gen_len, max_new=max_new).items()}
        outcome = torch.zeros((S, 4), dtype=torch.int32, device="cuda")
        bon = torch.zeros(B, dtype=torch.int32, device="cuda")
        _native.check(lib.sr_accept_commit(None, B, N, dev["seqs"].data_ptr(), dev["token_ids"].data_ptr(),
                                           dev["target"].data_ptr(), dev["tokens"].data_ptr(), stride,
                                           dev["seq_len"].data_ptr(), dev["gen_len"].data_ptr(),
                                           dev["max_new"].data_ptr(), bonus, outcome.data_ptr(),
                                           bon.data_ptr(), _native.stream_handle()), "accept")
        torch.cuda.synchronize()
        got_out, got_bon = outcome.cpu().numpy(), bon.cpu().numpy()
        got_tok, got_len = dev["tokens"].cpu().numpy(), dev["seq_len"].cpu().numpy()
        for b in range(B):
            rem = int(max_new[b] - gen_len[b])
            acc = []
            for n in range(N):
                q0, ql = seqs[b * N + n, 0], seqs[b * N + n, 1]
                if ql == 0 or rem <= 0:
                    acc.append(None)
                    continue
                nd, a = ql - 1, 0
                while a < nd and token_ids[q0 + a + 1] == target[q0 + a]:
                    a += 1
                acc.append((a, nd, q0))
            live = [(x[0], -n) for n, x in enumerate(acc) if x is not None]
            if not live:
                assert got_bon[b] == -1 and got_len[b] == seq_len[b]
                continue
            win = -max(live)[1]
            a, nd, q0 = acc[win]
            c = 1 if nd == 0 else (nd + bonus if a == nd else a + 1)
            c = min(c, rem)
            assert got_bon[b] == win
            assert got_len[b] == seq_len[b] + c
            assert got_tok[b, seq_len[b]:seq_len[b] + c].tolist() == target[q0:q0 + c].tolist()
            for n in range(N):
                row = got_out[b * N + n]
                if acc[n] is None:
                    assert row.tolist() == [0, 0, 0, 0]
                    continue
                an, ndn, _ = acc[n]
                exp_w = (0 if an == ndn else max(ndn - an - 1, 0)) if n == win else ndn
                assert row.tolist() == [ndn, an, c if n == win else 0, exp_w]


def test_synthetic_drafter_follows_reference_accept_law():
    """The reference-acceptance drafter accepts exactly the reference's
    `_verify_prefix` run (sim.py:977-981) on keyed draws, while the committed
    tokens stay the target's greedy output."""
    from oracle import rollout_oracle
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter
    from paper_2511_16193_b200.workload import gen_trace

    B, k, method = 4, 4, "draft-0.5b"
    s, w, m = make("tiny", "bf16", B=B)
    prompts = prompts_for(s.vocab, B, 6)
    reqs = gen_trace(scenarios.default_trace_spec(batch=B, seed=0))
    max_new = [70, 45, 90, 30]
    plain, _ = run_engine(m, prompts, max_new, k=0)
    truth = plain.outputs()
    eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(SyntheticDrafter(truth, reqs, method, 0),),
                        bonus_token=True, history=256)
    eng.prefill()
    steps = eng.run()
    assert eng.outputs() == truth
    rows = eng.outcome_rows(steps)
    for b, r in enumerate(reqs):
        u = rollout_oracle.accept_uniforms(0, r.id, method, max_new[b] + 8)
        p = r.latent_accept[method]
        g = 0
        for step in range(steps):
            n, a, c, _ = rows[step, b]
            if n == 0 and c == 0:
                continue
            exp_a = 0
            while exp_a < n and u[g + exp_a] < p:
                exp_a += 1
            assert a == exp_a, (b, step, g)
            g += c
        assert g == max_new[b]


def test_model_drafter_exactness_and_self_drafting():
    """K5 small-model drafter: a different drafter keeps outputs identical to
    plain decode; a drafter that *is* the target is accepted every time."""
    from paper_2511_16193_b200.engine import ModelDrafter, RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    B, k = 4, 4
    s, w, m = make("tiny", "bf16", B=B)
    prompts = prompts_for(s.vocab, B, 14)
    max_new = [40, 21, 33, 9]
    plain, _ = run_engine(m, prompts, max_new, k=0)

    def drafter(seed):
        d = DeviceModel(s, init_weights(s, seed=seed), dtype="bf16", max_requests=B, max_len=512,
                        max_tokens=512, max_seqs=B * 3)
        return ModelDrafter(d)

    other = RolloutEngine(m, prompts, max_new, k=k, drafters=(drafter(7),), history=256)
    other.prefill()
    other.run()
    assert other.outputs() == plain.outputs()

    selfd = RolloutEngine(m, prompts, max_new, k=k, drafters=(drafter(0),), history=256)
    selfd.prefill()
    steps = selfd.run()
    assert selfd.outputs() == plain.outputs()
    rows = selfd.outcome_rows(steps).reshape(-1, 4)
    live = rows[rows[:, 0] > 0]
    assert len(live) and (live[:, 1] == live[:, 0]).all()   # every draft accepted


def test_model_drafter_coupled_sampling():
    """T = 1: the drafter samples with the target's keyed Gumbel noise.  The
    output equals plain sampled decoding bit for bit; a drafter that is the
    target gets every draft accepted, a different one strictly fewer."""
    from paper_2511_16193_b200.engine import ModelDrafter, RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights

    B, k, T, seed = 4, 4, 1.0, 31
    s, w, m = make("tiny", "bf16", B=B)
    prompts = prompts_for(s.vocab, B, 14)
    max_new = [40, 21, 33, 9]
    from paper_2511_16193_b200.engine import NgramDrafter

    plain = RolloutEngine(m, prompts, max_new, k=0, drafters=(NgramDrafter(),), history=256,
                          temperature=T, seed=seed)
    plain.prefill()
    plain.run()

    def drafter(wseed):
        d = DeviceModel(s, init_weights(s, seed=wseed), dtype="bf16", max_requests=B, max_len=512,
                        max_tokens=512, max_seqs=B * 3)
        return ModelDrafter(d)

    rates = []
    for wseed in (0, 7):
        eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(drafter(wseed),), history=256,
                            temperature=T, seed=seed)
        eng.prefill()
        steps = eng.run()
        assert eng.outputs() == plain.outputs()
        rows = eng.outcome_rows(steps).reshape(-1, 4)
        live = rows[rows[:, 0] > 0]
        rates.append(live[:, 1].sum() / live[:, 0].sum())
    assert rates[0] == 1.0 and rates[1] < 1.0


def test_engine_outcomes_match_reference_coupled_golden():
    """Model-mode rollout (real tiny target, reference-acceptance drafter,
    w = k = 4, bonus off) reproduces the reference simulator's per-request
    VerificationOutcome stream (proposed, accepted, committed, wasted) of the
    config-1 golden run (tests/golden/sim_runs.json, c1-coupled-ngram-w4)."""
    from conftest import golden
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape
    from paper_2511_16193_b200.streams import stream
    from paper_2511_16193_b200.workload import gen_trace

    rec = next(r for r in golden("sim_runs.json") if r["name"] == "c1-coupled-ngram-w4")
    trace = gen_trace(scenarios.default_trace_spec(batch=8, seed=0))
    s = shape("tiny")
    prompts = [stream(0, r.id, "prompt").integers(0, s.vocab, size=r.prompt_len).astype(np.int32) for r in trace]
    lens = [r.true_len for r in trace]
    max_len = max(len(p) + L for p, L in zip(prompts, lens)) + 16
    m = DeviceModel(s, init_weights(s, seed=0), dtype="bf16", max_requests=8, max_len=max_len,
                    max_tokens=2048, max_seqs=24)
    plain = RolloutEngine(m, prompts, lens, k=0, history=1)
    plain.prefill()
    plain.run()
    truth = plain.outputs()
    eng = RolloutEngine(m, prompts, lens, k=4, drafters=(SyntheticDrafter(truth, trace, "ngram", 0),),
                        bonus_token=False, history=max(lens) + 1)
    eng.prefill()
    steps = eng.run()
    assert eng.outputs() == truth
    rows = eng.outcome_rows(steps)
    for b, r in enumerate(trace):
        got = [tuple(int(x) for x in row) for row in rows[:, b, :] if row[0] or row[2]]
        exp = [tuple(o[5:9]) for o in rec["outcomes"] if o[0] == r.id]
        assert got == exp, f"request {r.id}"


def test_decoupled_outcomes_match_reference_golden():
    """Depth-2 decoupled rollout (drafter and verifier roles; successors die
    with their rejected predecessor) reproduces the reference simulator's
    decoupled outcome stream, including depth-2 waste
    (tests/golden/sim_runs.json, c1-decoupled-ngram-w4, sim.py:1051-1092)."""
    from conftest import golden
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.decoupled import run_local
    from paper_2511_16193_b200.engine import RolloutEngine, SyntheticDrafter
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape
    from paper_2511_16193_b200.streams import stream
    from paper_2511_16193_b200.workload import gen_trace

    rec = next(r for r in golden("sim_runs.json") if r["name"] == "c1-decoupled-ngram-w4")
    trace = gen_trace(scenarios.default_trace_spec(batch=8, seed=0))
    s = shape("tiny")
    prompts = [stream(0, r.id, "prompt").integers(0, s.vocab, size=r.prompt_len).astype(np.int32) for r in trace]
    lens = [r.true_len for r in trace]
    max_len = max(len(p) + L for p, L in zip(prompts, lens)) + 16
    m = DeviceModel(s, init_weights(s, seed=0), dtype="bf16", max_requests=8, max_len=max_len,
                    max_tokens=2048, max_seqs=24)
    plain = RolloutEngine(m, prompts, lens, k=0, history=1)
    plain.prefill()
    plain.run()
    truth = plain.outputs()
    outs, rows = run_local(m, prompts, lens, 4, SyntheticDrafter(truth, trace, "ngram", 0))
    assert outs == truth
    for b, r in enumerate(trace):
        got = [tuple(int(x) for x in row) for row in rows[:, b, :] if row[0] or row[2]]
        exp = [tuple(o[5:9]) for o in rec["outcomes"] if o[0] == r.id]
        assert got == exp, f"request {r.id}"


@pytest.mark.parametrize("same_weights", [True, False])
def test_decoupled_small_model_drafter_equals_plain(same_weights):
    """K5 on the drafter side of decoupled mode (reference sim.py:860-917
    with a draft-model method): the drafter's context for window j+1 is the
    committed tokens plus in-flight window j.  With the target's own weights
    every verified window is fully accepted; with other weights windows are
    rejected and the drafter's KV cache rolls back to the corrected token.
    Both commit exactly the plain greedy sequence."""
    from paper_2511_16193_b200.decoupled import run_local
    from paper_2511_16193_b200.engine import ModelDrafter, RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel, init_weights

    B, k = 6, 4
    s, w, m = make("tiny", "bf16", B=B, max_len=256)
    prompts = prompts_for(s.vocab, B, 20)
    max_new = [30, 25, 40, 12, 33, 20]
    plain = RolloutEngine(m, prompts, max_new, k=0, history=1)
    plain.prefill()
    plain.run()
    truth = plain.outputs()
    dw = w if same_weights else init_weights(s, seed=5)
    dm = DeviceModel(s, dw, dtype="bf16", max_requests=B, max_len=256, max_tokens=B * (k + 2) * 4, max_seqs=B)
    outs, rows = run_local(m, prompts, max_new, k, ModelDrafter(dm))
    assert outs == truth
    live = rows[rows[:, :, 0] > 0]
    assert len(live) > 0
    full = (live[:, 1] == live[:, 0]).mean()
    if same_weights:
        assert full == 1.0
    else:
        assert full < 1.0


def test_decoupled_ngram_drafter_equals_plain():
    """The real n-gram drafter (K4) on the drafter side of decoupled mode:
    random prompts often give no proposal -- an empty window still commits
    the target's token (and discards its misaligned successor) -- and
    repetitive prompts give accepted drafts.  Output == plain greedy."""
    from paper_2511_16193_b200.decoupled import run_local
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    B, k = 6, 4
    s, w, m = make("tiny", "bf16", B=B, max_len=256)
    prompts = prompts_for(s.vocab, B, 21, alphabet=6)   # repetitive: n-gram matches
    prompts[0] = np.random.default_rng(3).integers(0, s.vocab, 30).astype(np.int32)  # no matches
    max_new = [20, 35, 40, 12, 33, 25]
    plain = RolloutEngine(m, prompts, max_new, k=0, history=1)
    plain.prefill()
    plain.run()
    truth = plain.outputs()
    outs, rows = run_local(m, prompts, max_new, k, NgramDrafter(1, 3))
    assert outs == truth
    assert int(rows[:, :, 1].clip(min=0).sum()) > 0      # some drafts accepted


def test_configs2_7b_shape_bon_ngram_and_model_drafters():
    """configs[2] widths (Qwen2.5-7B: H 3584, I 18944, 28/4 heads, G = 7), 2
    layers: Best-of-N with n-gram + small-model (0.5B-shaped) drafters commits
    exactly the plain greedy sequence."""
    from paper_2511_16193_b200.engine import ModelDrafter, NgramDrafter
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    B = 4
    s, w, m = make("qwen2.5-7b", "bf16", layers=2, B=B, branches=2 * B, max_len=512)
    prompts = prompts_for(min(s.vocab, 151936), B, 6)
    max_new = [40, 17, 29, 8]
    plain, _ = run_engine(m, prompts, max_new, k=0)
    ds = shape("qwen2.5-0.5b", 2)
    d = DeviceModel(ds, init_weights(ds, seed=3), dtype="bf16", max_requests=B, max_len=512,
                    max_tokens=512, max_seqs=B * 3)
    bon, steps = run_engine(m, prompts, max_new, k=4,
                            drafters=(NgramDrafter(1, 3), ModelDrafter(d), NgramDrafter(2, 4)))
    assert bon.outputs() == plain.outputs()


def test_configs4_32b_shape_sampled_bon4():
    """configs[4] widths (Qwen2.5-32B: H 5120, I 27648, 40/8 heads), 1 layer,
    T = 1 keyed sampling with Best-of-N N = 4: identical to plain sampling."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    B = 2
    s, w, m = make("qwen2.5-32b", "bf16", layers=1, B=2 * B, branches=3 * B, max_len=256)
    prompts = prompts_for(s.vocab, B, 10)
    max_new = [24, 13]

    def run(k, drafters):
        eng = RolloutEngine(m, prompts, max_new, k=k, drafters=drafters, history=128,
                            temperature=1.0, seed=44)
        eng.prefill()
        eng.run()
        return eng.outputs()

    plain = run(0, (NgramDrafter(),))
    assert run(4, (NgramDrafter(1, 3), NgramDrafter(2, 2), NgramDrafter(1, 1), NgramDrafter(3, 4))) == plain


def test_capture_io_step_matches_graph_step():
    """The host-facing step graph (H2D budgets -> step -> D2H results) advances
    the rollout exactly like the plain step graph and returns each step's
    outcome row and committed tokens."""
    import torch

    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    B, k = 4, 4
    s, w, m = make("tiny", "bf16", B=B)
    prompts = prompts_for(s.vocab, B, 20)
    max_new = [30, 30, 30, 30]
    a = RolloutEngine(m, prompts, max_new, k=k, drafters=(NgramDrafter(),), history=1)
    a.prefill()
    a.capture()
    b = RolloutEngine(m, prompts, max_new, k=k, drafters=(NgramDrafter(),), history=1)
    b.prefill()
    budget = torch.tensor(max_new, dtype=torch.int32).pin_memory()
    res = torch.zeros((B, 4 + k + 2), dtype=torch.int32).pin_memory()
    b.capture_io(budget, res)
    for _ in range(6):
        before = b.seq_len.clone()
        a.step()
        b.step_io()
        torch.cuda.synchronize()
        assert torch.equal(a.history[0], b.history[0])
        assert torch.equal(res[:, :4], b.history[0][:B].cpu())
        for r in range(B):
            c = int(res[r, 2])
            got = res[r, 4:4 + c].tolist()
            assert got == b.tokens[r, int(before[r]): int(before[r]) + c].tolist()
    assert a.outputs() == b.outputs()


def test_mixed_windows_per_request():
    """Request-level reconfiguration: one batch with per-request windows
    0..k (0 = plain decoding) commits the plain sequence and never proposes
    more than a request's window."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    B, k = 5, 4
    s, w, m = make("tiny", "bf16", B=B)
    prompts = prompts_for(s.vocab, B, 5)
    max_new = [40, 31, 27, 33, 19]
    plain, _ = run_engine(m, prompts, max_new, k=0)
    windows = [0, 1, 2, 3, 4]
    eng = RolloutEngine(m, prompts, max_new, k=k, drafters=(NgramDrafter(),), history=256)
    eng.set_windows(windows)
    eng.prefill()
    steps = eng.run()
    assert eng.outputs() == plain.outputs()
    rows = eng.outcome_rows(steps)
    for b, wb in enumerate(windows):
        assert int(rows[:, b, 0].max()) <= wb
    assert int(rows[:, 4, 0].max()) > 0   # the k = 4 request did speculate


def test_migrate_requests_between_engines():
    """Straggler pull / tail rebalancing as data movement: requests moved
    mid-rollout (token row, lengths, KV pages) into other slots of another
    engine continue to exactly the plain-decoding output."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine
    from paper_2511_16193_b200.migrate import migrate_local
    from paper_2511_16193_b200.model import DeviceModel

    B = 4
    s, w, m1 = make("tiny", "bf16", B=B)
    m2 = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=512, max_tokens=512, max_seqs=B * 3)
    prompts = prompts_for(s.vocab, B, 8)
    max_new = [50, 41, 37, 45]
    plain, _ = run_engine(m1, prompts, max_new, k=0)
    src = RolloutEngine(m1, prompts, max_new, k=4, drafters=(NgramDrafter(),), history=64)
    src.prefill()
    for _ in range(5):
        src.step()
    perm = [2, 0, 3, 1]                       # source slot b -> destination slot perm[b]
    dprompts = [None] * B
    for b in range(B):
        dprompts[perm[b]] = prompts[b]
    dmax = [0] * B
    for b in range(B):
        dmax[perm[b]] = max_new[b]
    dst = RolloutEngine(m2, dprompts, dmax, k=4, drafters=(NgramDrafter(),), history=64)
    dst.prefill()
    moved = sum(migrate_local(src, b, dst, perm[b]) for b in range(B))
    assert moved > 0 and src.done()
    dst.run()
    out = dst.outputs()
    assert [out[perm[b]] for b in range(B)] == plain.outputs()


def test_migrate_into_smaller_engine_rejected():
    """A destination slot must hold the request's whole remaining budget, not
    only its current length (a long straggler moved into an engine
    sized for shorter requests would write past its token row)."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine
    from paper_2511_16193_b200.errors import ConfigError
    from paper_2511_16193_b200.migrate import migrate_local

    s, w, m = make("tiny", "bf16", B=4)
    prompts = prompts_for(s.vocab, 2, 8, lo=30, hi=31)
    src = RolloutEngine(m, prompts[:1], [120], k=4, drafters=(NgramDrafter(),), history=8)
    src.prefill()
    src.step()
    dst = RolloutEngine(m, prompts[1:], [8], k=4, drafters=(NgramDrafter(),), history=8)
    with pytest.raises(ConfigError):
        migrate_local(src, 0, dst, 0)
    assert not src.done()           # a refused move leaves the source untouched


def test_migrate_updates_slot_state_and_budget_cap():
    """Unpack follows the new occupant: prompt length (outputs() slicing), the
    slot capacity, a model drafter's cache; the retired source slot stays
    retired even when the host-facing graph copies the old budgets in."""
    from paper_2511_16193_b200.engine import ModelDrafter, NgramDrafter, RolloutEngine
    from paper_2511_16193_b200.migrate import migrate_local
    from paper_2511_16193_b200.model import DeviceModel

    B = 2
    s, w, m1 = make("tiny", "bf16", B=B)
    m2 = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=512, max_tokens=512, max_seqs=B * 3)
    md = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=512, max_tokens=512, max_seqs=B * 3)
    prompts = prompts_for(s.vocab, 4, 12)
    max_new = [60, 55]
    plain, _ = run_engine(m1, prompts[:2], max_new, k=0)
    src = RolloutEngine(m1, prompts[:2], max_new, k=4, drafters=(NgramDrafter(),), history=1)
    src.prefill()
    budget_h = torch.tensor(max_new, dtype=torch.int32).pin_memory()
    res_h = torch.zeros((B, 4 + 6), dtype=torch.int32).pin_memory()
    g = src.capture_io(budget_h, res_h)
    for _ in range(3):
        src.step_io(g)
    # destination: other prompts (different lengths) and a model drafter that
    # uses the target's own weights (drafts == target tokens once in sync)
    dst = RolloutEngine(m2, prompts[2:], [70, 70], k=4, drafters=(ModelDrafter(md),), history=64)
    dst.prefill()
    migrate_local(src, 1, dst, 0)
    torch.cuda.synchronize()
    assert dst.prompt_lens[0] == len(prompts[1])
    for _ in range(4):              # host budgets copied in again: slot 1 must not revive
        src.step_io(g)
    torch.cuda.synchronize()
    assert int(src.gen_len[1]) == int(src.max_new[1]) == int(src.max_new_cap[1])
    steps = dst.run()
    assert dst.outputs()[0] == plain.outputs()[1]
    rows = dst.outcome_rows(steps)
    # the re-prefilled drafter cache proposes the target's tokens: windows accept
    assert rows[:, 0, 1].sum() > 0.8 * rows[:, 0, 0].sum()


def test_capture_io_budget_clamped_to_capacity():
    """A host budget above the constructor's max_new is clamped on device."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    s, w, m = make("tiny", "bf16", B=2)
    prompts = prompts_for(s.vocab, 2, 13)
    eng = RolloutEngine(m, prompts, [9, 5], k=4, drafters=(NgramDrafter(),), history=1)
    eng.prefill()
    budget_h = torch.tensor([10_000, 10_000], dtype=torch.int32).pin_memory()
    res_h = torch.zeros((2, 4 + 6), dtype=torch.int32).pin_memory()
    g = eng.capture_io(budget_h, res_h)
    for _ in range(30):
        eng.step_io(g)
    torch.cuda.synchronize()
    assert eng.gen_len.tolist() == [9, 5]


def test_prefill_prompts_longer_than_max_tokens():
    """Chunked prefill: prompts longer than the model's max_tokens are split
    into pieces; decoding afterwards matches a model that prefilled them whole."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine
    from paper_2511_16193_b200.model import DeviceModel

    B = 2
    s, w, big = make("tiny", "bf16", B=B, max_tokens=1024)
    small = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=512, max_tokens=64, max_seqs=B * 3)
    prompts = prompts_for(s.vocab, B, 9, lo=150, hi=300)
    max_new = [20, 17]
    outs = []
    for m in (big, small):
        e = RolloutEngine(m, prompts, max_new, k=0, drafters=(NgramDrafter(),), history=1)
        e.prefill()
        e.run()
        outs.append(e.outputs())
    assert outs[0] == outs[1]


@pytest.mark.parametrize("k", [1, 2, 8])
def test_edge_cases_spec_equals_plain(k):
    """Ragged and degenerate batches: zero-budget requests (empty output),
    one-token prompts, prompts ending on either side of a 64-token page
    boundary, budgets that end mid-window, and window sizes 1 / 2 / 8 --
    speculative output equals plain decoding and zero-budget requests
    commit nothing."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    B = 8
    s, w, m = make("tiny", "bf16", B=B, max_len=512)
    rng = np.random.default_rng(11)
    words = rng.integers(0, s.vocab, size=12)
    plens = [1, 63, 64, 65, 127, 128, 2, 200]
    prompts = [words[rng.integers(0, 12, size=L)].astype(np.int32) for L in plens]
    max_new = [0, 5, 1, 64, 0, 33, 70, k + 1]
    plain = RolloutEngine(m, prompts, max_new, k=0, history=1)
    plain.prefill()
    plain.run()
    ref = plain.outputs()
    assert ref[0] == [] and ref[4] == []
    assert [len(r) for r in ref] == max_new
    spec = RolloutEngine(m, prompts, max_new, k=k, drafters=(NgramDrafter(1, 3),), history=1)
    spec.prefill()
    spec.run()
    assert spec.outputs() == ref


@pytest.mark.parametrize("N", [1, 3])
def test_compacted_batch_equals_fixed_layout(N):
    """Live-row compaction (sr_build_verify_batch live_rows): finished
    requests and unproposed draft slots take no rows and the GEMMs skip the
    dead tiles; outputs, outcome rows and the per-step live-row count equal
    the fixed-layout batch's."""
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine

    B, k = 6, 4
    s, w, m = make("tiny", "bf16", B=B, branches=B * (N - 1), max_len=256)
    prompts = prompts_for(s.vocab, B, 31, alphabet=8)
    max_new = [3, 40, 17, 29, 1, 35]          # requests finish at different steps
    drafters = tuple(NgramDrafter(1 + i, 3 + i) for i in range(N))
    res = []
    for compact in (False, True):
        eng = RolloutEngine(m, prompts, max_new, k=k, drafters=drafters, history=256, compact=compact)
        eng.prefill()
        live, steps = [], 0
        while not eng.done():
            eng.step()
            steps += 1
            sq = eng.seqs.cpu().numpy()
            live.append((int(eng.live_rows.item()), int(sq[:, 1].sum())))
        res.append((eng.outputs(), eng.outcome_rows(steps), live))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])
    for got, total in res[1][2]:
        assert got == total                    # packed rows == sum of window lengths
    assert res[1][2][-1][0] < B * N * (k + 1)  # the tail ran on fewer rows


def test_pack_results_rejects_pageable_host_buffer():
    """sr_pack_results writes device or pinned host memory (zero-copy D2H); a
    pageable host buffer is a config error, not a device fault."""
    from paper_2511_16193_b200 import _native

    lib = _native.lib()
    B, N, w = 4, 1, 6
    outcome = torch.zeros((B, 4), dtype=torch.int32, device="cuda")
    tokens = torch.zeros((B, 32), dtype=torch.int32, device="cuda")
    seq_before = torch.ones(B, dtype=torch.int32, device="cuda")
    pageable = torch.zeros((B, 4 * N + w), dtype=torch.int32)
    rc = lib.sr_pack_results(B, N, w, outcome.data_ptr(), tokens.data_ptr(), 32, seq_before.data_ptr(),
                             pageable.data_ptr(), _native.stream_handle())
    assert rc == 2
    pinned = pageable.pin_memory()
    tokens[:, 1:7] = torch.arange(6, dtype=torch.int32, device="cuda")
    outcome[:, 0] = 3
    _native.check(lib.sr_pack_results(B, N, w, outcome.data_ptr(), tokens.data_ptr(), 32, seq_before.data_ptr(),
                                      pinned.data_ptr(), _native.stream_handle()), "pack")
    torch.cuda.synchronize()
    assert pinned[:, 0].tolist() == [3] * B and pinned[0, 4:].tolist() == list(range(6))
