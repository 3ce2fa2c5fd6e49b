"""Model-mode speculative rollout on one GPU (the hot path of BASELINE.json).

One :meth:`RolloutEngine.step` is one speculation window for every live
request of the batch, entirely on device:

    sr_ngram_propose      K4  n-gram drafts from the token buffer
    sr_build_verify_batch     verify rows [last token, d_1..d_k] per drafter
    sr_model_forward      K1+K2+K6  target verify forward, fused argmax
    sr_accept_commit      K3  accepted prefix, Best-of-N select, commit, and
                              the winning branch's KV -> paged cache (N > 1)

This replaces one ``_Executor.begin_round``/``end_round`` pair of the
reference (``sim.py:834-1092``) with real drafting and verification; the
outcome rows carry the reference's ``VerificationOutcome`` fields.  The step
needs no host synchronization; the host only reads outcome rows when asked.
Steps can be captured into a CUDA graph (:meth:`capture`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import ConfigError
from .model import DeviceModel, seq_table


@dataclass(frozen=True)
class NgramDrafter:
    """vLLM-style prompt-lookup drafter (``ngram_proposer.py:198-285``)."""

    min_n: int = 1
    max_n: int = 3
    name: str = "ngram"


@dataclass(frozen=True)
class PooledNgramDrafter:
    """Prompt lookup over the whole batch (``sr_pooled_ngram_propose``): the
    request's own context first, then the other requests' committed tokens
    (RL groups sample one prompt several times).  Equals :class:`NgramDrafter`
    for a single request."""

    min_n: int = 1
    max_n: int = 3
    name: str = "pooled-ngram"


class SyntheticDrafter:
    """Drafter whose acceptance follows the reference's keyed Bernoulli law.

    ``truth[b]`` is the target model's greedy continuation of request b
    (from a plain-decode pass), ``method`` names the reference acceptance
    stream: draft token g is the true token iff
    ``stream(seed, rid, "accept_draw", method, g // 256).random(256)[g % 256]
    < latent_accept[method]`` (``sim.py:322-336``), generated on device by
    ``sr_keyed_uniforms``.
    """

    name = "synthetic"

    def __init__(self, truth: list[list[int]], requests, method: str, seed: int, device="cuda",
                 vocab: int = 0, capacity: int = 0):
        from .verify import CHUNK, entropy_words, keyed_fill

        B = len(truth)
        L = max(max(len(t) for t in truth), capacity)  # capacity: rows for adopted requests
        chunks = max(1, math.ceil(L / CHUNK))
        self.stride = chunks * CHUNK
        tt = np.zeros((B, self.stride), dtype=np.int32)
        for b, t in enumerate(truth):
            tt[b, : len(t)] = t
        self.truth = torch.from_numpy(tt).to(device)
        self.truth_len = torch.tensor([len(t) for t in truth], dtype=torch.int32, device=device)
        self.uniforms = torch.empty((B, self.stride), dtype=torch.float64, device=device)
        keyed_fill("uniforms", [entropy_words(seed, r.id, "accept_draw", method, c)
                                for r in requests for c in range(chunks)], CHUNK, self.uniforms)
        self.p = torch.tensor([r.latent_accept[method] for r in requests], dtype=torch.float64,
                              device=device)
        self.method = method
        self.vocab = vocab


# the drafter's own sampling stream in rejection mode (independent of the
# target's keyed noise, which would couple the two samples)
DRAFT_SEED_SALT = 0x6A09E667


class ModelDrafter:
    """Small-model drafter (K5; reference methods ``draft-0.5b``/``draft-1.5b``,
    ``scenarios.py:25-29``): k decode steps of its own decoder per window,
    with its own paged KV cache.  Each window first catches the drafter's
    cache up on the tokens committed since the previous window
    (``sr_draft_model_batch`` step 0), then decodes k-1 more tokens.

    Under a sampled target (engine temperature T > 0) the drafter samples
    with the *same* keyed Gumbel noise (seed, request, position) at the same
    T: Gumbel-coupled speculative sampling.  Every committed token is the
    target's keyed sample, so the output equals plain sampled decoding bit
    for bit, and a draft is accepted exactly when the two models' perturbed
    argmaxes agree (probability -> 1 as q -> p).

    With ``RolloutEngine(acceptance="rejection")`` the drafter instead
    samples its window from q with its own keyed stream and keeps q's logit
    rows; K3 then runs Leviathan rejection sampling (``sr_accept_rejection``):
    outputs follow the target's distribution (not its keyed sample), and a
    draft is accepted with probability sum_v min(p_v, q_v), the maximum any
    coupling reaches.  Its DeviceModel needs ``logits_capacity >= batch``."""

    name = "model"

    def __init__(self, model: DeviceModel, name: str = "draft-0.5b"):
        self.m = model
        self.name = name
        self.eng = None

    def attach(self, eng: "RolloutEngine") -> None:
        B, k, dev = eng.B, eng.k, eng.dev
        if self.m.max_tokens < B * (k + 2) or self.m.max_seqs < B or self.m.max_len < eng.max_key + 2:
            raise ConfigError("drafter model capacity too small for the batch")
        self.eng = eng
        self.dkv_len = torch.tensor([L - 1 for L in eng.prompt_lens], dtype=torch.int32, device=dev)
        self.token_ids = torch.zeros(B * (k + 2), dtype=torch.int32, device=dev)
        self.positions = torch.zeros(B * (k + 2), dtype=torch.int32, device=dev)
        self.seqs = torch.zeros((B, 8), dtype=torch.int32, device=dev)
        self.logit_rows = torch.zeros(B, dtype=torch.int32, device=dev)
        self.out = torch.zeros(B, dtype=torch.int32, device=dev)
        prefill_model(self.m, eng.tokens, [L - 1 for L in eng.prompt_lens])

    def reset_slot(self, b: int) -> None:
        """Rebuild slot ``b``'s drafter cache from the engine's token row (a
        request was migrated into it): KV of [0, seq_len - 1), the catch-up
        step then feeds the last committed token."""
        L = int(self.eng.seq_len[b])
        if L > 1:
            prefill_model(self.m, self.eng.tokens, {b: L - 1})
        self.dkv_len[b] = L - 1

    def enqueue(self, drafts, ndraft) -> None:
        e, lib, st = self.eng, self.eng.lib, _native.stream_handle()
        rejection = e.acceptance == "rejection"
        if rejection and not hasattr(self, "q_logits"):
            if self.m.desc.logits_capacity < e.B:
                raise ConfigError("rejection sampling: the drafter model needs logits_capacity >= batch")
            self.q_logits = torch.empty((e.k, e.B, self.m.s.vocab), dtype=torch.float32, device=e.dev)
            self.key_req = torch.arange(e.B, dtype=torch.int32, device=e.dev)
            self.key_pos = torch.zeros(e.B, dtype=torch.int32, device=e.dev)
        for step in range(e.k + 1):
            _native.check(lib.sr_draft_model_batch(
                e.B, e.k, step, e.tokens.data_ptr(), e.stride, e.seq_len.data_ptr(), e.gen_len.data_ptr(),
                e.max_new.data_ptr(), self.dkv_len.data_ptr(), self.out.data_ptr(), drafts.data_ptr(),
                ndraft.data_ptr(), self.token_ids.data_ptr(), self.positions.data_ptr(), self.seqs.data_ptr(),
                self.logit_rows.data_ptr(), self.key_pos.data_ptr() if rejection else None, st),
                "sr_draft_model_batch")
            if step == e.k:
                break
            # step 0: catch-up rows [b*(k+2), +k+2), logits at each request's
            # last one; steps >= 1: one decode row per request, rows [0, B)
            rows = (self.token_ids, self.positions, self.logit_rows, e.k + 2) if step == 0 else \
                (self.token_ids[:e.B], self.positions[:e.B], None, 1)
            if rejection:
                # the drafter samples its window from q = softmax(logits / T)
                # with its own keyed noise, and keeps q's rows for K3
                q = self.q_logits[step]
                self.m.forward(rows[0], rows[1], self.seqs, num_seqs=e.B, max_q_len=rows[3],
                               max_key=e.max_key, out=q, logit_rows=rows[2], output=1)
                _native.check(lib.sr_sample_rows(
                    q.data_ptr(), e.B, q.shape[1], q.shape[1], self.key_req.data_ptr(), self.key_pos.data_ptr(),
                    (e.seed ^ DRAFT_SEED_SALT) & 0xFFFFFFFF, e.temperature, self.out.data_ptr(), st),
                    "sr_sample_rows")
            else:
                self.m.forward(rows[0], rows[1], self.seqs, num_seqs=e.B, max_q_len=rows[3],
                               max_key=e.max_key, out=self.out, logit_rows=rows[2], output=e._out_mode,
                               temperature=e.temperature, seed=e.seed)


def prefill_model(m: DeviceModel, tokens, lens) -> None:
    """Chunked prompt forward writing KV for positions [0, lens[b]) of every
    request b into ``m``'s paged cache (the logits are not needed).  ``lens``
    is a list over all slots or a ``{slot: length}`` dict (re-prefill of
    single slots).  Prompts longer than the model's ``max_tokens`` are split
    into pieces; a piece attends to its request's earlier pieces through the
    cache."""
    dev = tokens.device
    pieces = []
    for b, L in (lens.items() if isinstance(lens, dict) else enumerate(lens)):
        off = 0
        while off < L:
            n = min(m.max_tokens, L - off)
            pieces.append((b, off, n))
            off += n
    i = 0
    while i < len(pieces):
        rows, tok_rows, pos_rows = [], [], []
        start, max_q, max_key = 0, 0, 0
        while i < len(pieces):
            b, off, n = pieces[i]
            if rows and (start + n > m.max_tokens or len(rows) + 1 > m.max_prefill_seqs(max(max_q, n))):
                break
            rows.append((start, n, b, off, -1))
            tok_rows.append(tokens[b, off:off + n])
            pos_rows.append(torch.arange(off, off + n, dtype=torch.int32, device=dev))
            start += n
            max_q = max(max_q, n)
            max_key = max(max_key, off + n - 1)
            i += 1
        lr = torch.tensor([r[0] + r[1] - 1 for r in rows], dtype=torch.int32, device=dev)
        out = torch.empty(len(rows), dtype=torch.int32, device=dev)
        m.forward(torch.cat(tok_rows), torch.cat(pos_rows), seq_table(rows, dev), num_seqs=len(rows),
                  max_q_len=max_q, max_key=max_key, out=out, logit_rows=lr)


class RolloutEngine:
    """Batch state (token buffer, lengths, budgets) + per-step device work."""

    def __init__(self, target: DeviceModel, prompts: list[np.ndarray], max_new: list[int], *, k: int = 4,
                 drafters: tuple = (NgramDrafter(),), bonus_token: bool = False, history: int = 0,
                 temperature: float = 0.0, seed: int = 0, acceptance: str = "exact", compact: bool = True,
                 capacity: int = 0):
        if not prompts:
            raise ConfigError("empty batch")
        if len(prompts) != len(max_new):
            raise ConfigError("prompts / max_new length mismatch")
        self.m = target
        self.lib = target.lib
        self.dev = target.dev
        self.k = k
        self.drafters = tuple(drafters)
        self.N = len(self.drafters)
        self.B = len(prompts)
        self.bonus = 1 if bonus_token else 0
        # T = 0: greedy; T > 0: keyed Gumbel-max sampling (exact match still
        # verifies because the target's draw is keyed by (seed, request, position))
        self.temperature, self.seed = float(temperature), int(seed)
        self._out_mode = 2 if self.temperature > 0 else 0
        # acceptance rule: "exact" -- exact match against the target's token
        # (greedy, or its keyed sample at T > 0; every committed token equals
        # plain decoding's), or "rejection" -- Leviathan rejection sampling
        # for one stochastic model drafter (distribution-preserving)
        if acceptance not in ("exact", "rejection"):
            raise ConfigError(f"acceptance must be 'exact' or 'rejection', not {acceptance!r}")
        self.acceptance = acceptance
        if acceptance == "rejection":
            if self.N != 1 or not isinstance(self.drafters[0], ModelDrafter):
                raise ConfigError("rejection sampling needs exactly one model drafter (N = 1)")
            if self.temperature <= 0:
                raise ConfigError("rejection sampling needs temperature > 0")
            if self.drafters[0].m.s.vocab != target.s.vocab:
                raise ConfigError("rejection sampling needs drafter and target over the same vocabulary")
            if target.desc.logits_capacity < self.B * (k + 1):
                raise ConfigError("rejection sampling: the target needs logits_capacity >= B * (k + 1)")
        if self.N > 1 and target.branches < self.B * (self.N - 1):
            raise ConfigError("target model needs max_branches >= B*(N-1) for Best-of-N")
        if self.B * self.N > target.max_seqs or self.B * self.N * (k + 1) > target.max_tokens:
            raise ConfigError("batch exceeds the model's max_seqs / max_tokens")
        lens = [len(p) for p in prompts]
        # capacity: positions per slot beyond this batch's own needs (a rank
        # that adopts migrated stragglers sizes its slots for the whole job)
        need = max(max(l + n for l, n in zip(lens, max_new)), capacity) + k + 2
        if need > target.max_len:
            raise ConfigError(f"prompt + generation ({need}) exceeds model max_len {target.max_len}")
        self.stride = int(math.ceil(need / 16) * 16)
        dev = self.dev
        tok = np.zeros((self.B, self.stride), dtype=np.int32)
        for i, p in enumerate(prompts):
            tok[i, : len(p)] = p
        self.prompt_lens = lens
        self.tokens = torch.from_numpy(tok).to(dev)
        self.seq_len = torch.tensor(lens, dtype=torch.int32, device=dev)
        self.gen_len = torch.zeros(self.B, dtype=torch.int32, device=dev)
        self.max_new = torch.tensor(max_new, dtype=torch.int32, device=dev)
        # capacity of each slot (its token row / KV pages were sized for it):
        # every step clamps max_new to it on device, so host budgets copied in
        # by capture_io cannot overflow a row, and retire() is permanent
        self.max_new_cap = self.max_new.clone()
        S, R = self.B * self.N, self.B * self.N * (k + 1)
        self.drafts = torch.full((self.N, self.B, k), -1, dtype=torch.int32, device=dev)
        self.ndraft = torch.zeros((self.N, self.B), dtype=torch.int32, device=dev)
        self.ngram_scratch = torch.zeros(2 * self.B, dtype=torch.int64, device=dev)
        self.token_ids = torch.zeros(R, dtype=torch.int32, device=dev)
        self.positions = torch.zeros(R, dtype=torch.int32, device=dev)
        self.seqs = torch.zeros((S, 8), dtype=torch.int32, device=dev)
        self.target_ids = torch.zeros(R, dtype=torch.int32, device=dev)
        self.history = torch.zeros((max(history, 1), S, 4), dtype=torch.int32, device=dev)
        self.bon = torch.zeros(self.B, dtype=torch.int32, device=dev)
        # per-request window caps (request-level reconfiguration, reference
        # planner.reconfigure / sim.py:445-510): one batch mixes windows
        # 0..k; rows beyond a request's window are simply not verified
        self.window = torch.full((self.B,), k, dtype=torch.int32, device=dev)
        # live-row compaction: each step packs only live rows (finished
        # requests, gap rounds and unproposed draft slots take none) and the
        # forward's GEMMs skip the dead tiles (sr_build_verify_batch live_rows)
        self.compact = bool(compact)
        # Best-of-N drafter assignment: drafter n proposes for request b only
        # where active[n, b] != 0 (all on by default; policy.RolloutDriver
        # turns extra drafters on for tail requests when the batch drains)
        self.active = torch.ones((self.N, self.B), dtype=torch.int32, device=dev)
        self.live_rows = torch.zeros(1, dtype=torch.int32, device=dev)
        if acceptance == "rejection":
            self.p_logits = torch.empty((R, target.s.vocab), dtype=torch.float32, device=dev)
            # per verify row (lse_p, lse_q, log p(d), log q(d)) + per-request chunk partials
            self.rs_stats = torch.zeros(int(_native.lib().sr_accept_rejection_workspace_floats(self.B, k)),
                                        dtype=torch.float32, device=dev)
        self.steps = 0
        self.max_key = need - 1
        self.graph = None

    # -- prefill -------------------------------------------------------------

    def prefill(self) -> None:
        """Cache the KV of every prompt token but the last.  The last prompt
        token is the "last committed token" the first window starts from, so
        generated position 0 comes out of the first verify window -- the
        reference's round structure, where every output token is produced by
        a window (``sim.py:834-928``).  Model drafters prefill their caches."""
        prefill_model(self.m, self.tokens, [L - 1 for L in self.prompt_lens])
        for d in self.drafters:
            if isinstance(d, ModelDrafter):
                d.attach(self)

    # -- one speculation window ------------------------------------------------

    def _side_stream(self, n: int):
        if not hasattr(self, "_sides"):
            self._sides = {}
        if n not in self._sides:
            self._sides[n] = torch.cuda.Stream(device=self.dev)
        return self._sides[n]

    def _enqueue_step(self, slot: int) -> None:
        lib, st = self.lib, _native.stream_handle()
        drafts_ptr, nd_ptr = None, None
        if self.k > 0:
            # several small-model drafters (Best-of-N) are independent small-M
            # forwards that each fill a fraction of the GPU: run them on their
            # own streams (graph branches) and join before the verify batch
            cur = torch.cuda.current_stream()
            parallel = sum(isinstance(d, ModelDrafter) for d in self.drafters) > 1
            forks = []
            for n, d in enumerate(self.drafters):
                if isinstance(d, ModelDrafter):
                    if parallel:
                        side = self._side_stream(n)
                        side.wait_stream(cur)
                        with torch.cuda.stream(side):
                            d.enqueue(self.drafts[n], self.ndraft[n])
                        forks.append(side)
                    else:
                        d.enqueue(self.drafts[n], self.ndraft[n])
                    continue
                if isinstance(d, SyntheticDrafter):
                    _native.check(lib.sr_synthetic_draft(
                        self.B, self.k, d.truth.data_ptr(), d.stride, d.truth_len.data_ptr(),
                        d.uniforms.data_ptr(), d.stride, d.p.data_ptr(), self.gen_len.data_ptr(),
                        d.vocab or self.m.s.vocab, self.drafts[n].data_ptr(), self.ndraft[n].data_ptr(), st),
                        "sr_synthetic_draft")
                    continue
                propose = lib.sr_pooled_ngram_propose if isinstance(d, PooledNgramDrafter) else lib.sr_ngram_propose
                _native.check(propose(
                    self.B, self.tokens.data_ptr(), self.stride, self.seq_len.data_ptr(), d.min_n, d.max_n,
                    self.k, self.drafts[n].data_ptr(), self.ndraft[n].data_ptr(),
                    self.ngram_scratch.data_ptr(), st), "ngram propose")
            for side in forks:
                cur.wait_stream(side)
            drafts_ptr, nd_ptr = self.drafts.data_ptr(), self.ndraft.data_ptr()
        _native.check(lib.sr_build_verify_batch(
            self.B, self.N, self.k, self.tokens.data_ptr(), self.stride, self.seq_len.data_ptr(),
            self.gen_len.data_ptr(), self.max_new.data_ptr(), self.max_new_cap.data_ptr(), drafts_ptr, nd_ptr,
            self.window.data_ptr(), self.active.data_ptr() if self.N > 1 else None,
            self.token_ids.data_ptr(), self.positions.data_ptr(), self.seqs.data_ptr(),
            self.live_rows.data_ptr() if self.compact else None, st),
            "sr_build_verify_batch")
        out = self.history[slot]
        if self.acceptance == "rejection":
            d = self.drafters[0]
            self.m.forward(self.token_ids, self.positions, self.seqs, num_seqs=self.B, max_q_len=self.k + 1,
                           max_key=self.max_key, out=self.p_logits, output=1, live_rows=self._live())
            V = self.p_logits.shape[1]
            _native.check(lib.sr_accept_rejection(
                self.B, self.k, self.seqs.data_ptr(), self.token_ids.data_ptr(), self.p_logits.data_ptr(), V,
                d.q_logits.data_ptr() if self.k else None, V, V, self.temperature, self.seed & 0xFFFFFFFF,
                self.tokens.data_ptr(), self.stride, self.seq_len.data_ptr(), self.gen_len.data_ptr(),
                self.max_new.data_ptr(), self.bonus, self.rs_stats.data_ptr(), out.data_ptr(), self.bon.data_ptr(),
                st), "sr_accept_rejection")
            return
        self.m.forward(self.token_ids, self.positions, self.seqs, num_seqs=self.B * self.N,
                       max_q_len=self.k + 1, max_key=self.max_key, out=self.target_ids,
                       output=self._out_mode, temperature=self.temperature, seed=self.seed,
                       live_rows=self._live())
        _native.check(lib.sr_accept_commit(
            self.m.handle, self.B, self.N, self.seqs.data_ptr(), self.token_ids.data_ptr(),
            self.target_ids.data_ptr(), self.tokens.data_ptr(), self.stride, self.seq_len.data_ptr(),
            self.gen_len.data_ptr(), self.max_new.data_ptr(), self.bonus, out.data_ptr(), self.bon.data_ptr(), st),
            "sr_accept_commit")

    def _live(self):
        return self.live_rows if self.compact else None

    def step(self) -> None:
        slot = self.steps % self.history.shape[0]
        if self.graph is not None and slot == 0:
            self.graph.replay()
        else:
            self._enqueue_step(slot)
        self.steps += 1

    def capture(self, install: bool = True):
        """Capture one step (history slot 0) into a CUDA graph; ``install``
        makes :meth:`step` replay it."""
        if self.history.shape[0] != 1:
            raise ConfigError("graph capture needs history=0/1 (the graph writes slot 0)")
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g.capture_begin()
            self._enqueue_step(0)
            g.capture_end()
        torch.cuda.current_stream().wait_stream(s)
        if install:
            self.graph = g
        return g

    def capture_io(self, budget_host: torch.Tensor, result_host: torch.Tensor):
        """Host-facing step as one CUDA graph: H2D of the per-request budgets
        (``budget_host``, pinned int32 [B]), the speculation step, and D2H of
        each request's N drafter outcome rows and its next k+2 token slots
        (``result_host``, pinned int32 [B, 4 * N + k + 2]).  Budgets are clamped
        on device to the constructor's ``max_new`` (:attr:`max_new_cap`): a
        larger host budget cannot grow a request past its slot.  :meth:`step_io`
        replays the latest one (or pass the returned graph); the caller waits
        for the step (synchronize or an event recorded after the replay)
        before reading ``result_host``.  Capturing two graphs over two result
        buffers lets a host loop read step i while step i+1 runs."""
        if self.history.shape[0] != 1:
            raise ConfigError("graph capture needs history=0/1 (the graph writes slot 0)")
        w = self.k + 2
        cols = 4 * self.N + w
        if tuple(result_host.shape) != (self.B, cols) or budget_host.numel() != self.B:
            raise ConfigError("result_host must be [B, 4 * N + k + 2] and budget_host [B]")
        if not (budget_host.is_pinned() and result_host.is_pinned()):
            raise ConfigError("capture_io needs pinned host buffers (tensor.pin_memory())")
        if budget_host.dtype != torch.int32 or result_host.dtype != torch.int32 or not result_host.is_contiguous():
            raise ConfigError("capture_io buffers are contiguous int32")
        seq_before = torch.empty_like(self.seq_len)
        if not hasattr(self, "_io_keep"):
            self._io_keep = []
        self._io_keep.append((seq_before, budget_host, result_host))   # buffers the graph reads/writes stay alive
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g.capture_begin()
            # H2D of the budgets and D2H of the results are zero-copy kernel
            # accesses to the pinned buffers: no copy-engine nodes in the graph
            _native.check(self.lib.sr_io_begin(
                self.B, budget_host.data_ptr(), self.max_new.data_ptr(), self.seq_len.data_ptr(),
                seq_before.data_ptr(), _native.stream_handle()), "sr_io_begin")
            self._enqueue_step(0)
            _native.check(self.lib.sr_pack_results(
                self.B, self.N, w, self.history[0].data_ptr(), self.tokens.data_ptr(), self.stride,
                seq_before.data_ptr(), result_host.data_ptr(), _native.stream_handle()), "sr_pack_results")
            g.capture_end()
        torch.cuda.current_stream().wait_stream(s)
        self.graph_io = g
        return g

    def step_io(self, graph=None) -> None:
        (graph or self.graph_io).replay()
        self.steps += 1

    def set_active(self, mask) -> None:
        """Best-of-N drafter assignment: ``mask`` [N, B] (nonzero = drafter n
        proposes for request b).  Drafter 0 (the incumbent) stays on.  In
        place, so captured step graphs pick it up."""
        a = torch.as_tensor(mask, dtype=torch.int32)
        if a.shape != (self.N, self.B):
            raise ConfigError(f"active mask must be [{self.N}, {self.B}]")
        a = a.clone()
        a[0] = 1
        self.active.copy_(a.to(self.dev))

    def retire(self, b: int) -> None:
        """Stop request ``b`` where it is (its slot was migrated away): budget
        and capacity both drop to the generated length, so no later host
        budget revives it."""
        self.max_new[b] = self.gen_len[b]
        self.max_new_cap[b] = self.gen_len[b]

    def set_windows(self, windows) -> None:
        """Per-request window caps in [0, k] (0 = plain decoding for that
        request), e.g. the windows of ``planner.reconfigure``'s request plans.
        In place, so captured step graphs pick them up."""
        w = torch.as_tensor(windows, dtype=torch.int32)
        if w.shape != (self.B,) or int(w.min()) < 0 or int(w.max()) > self.k:
            raise ConfigError(f"windows must be {self.B} values in [0, {self.k}]")
        self.window.copy_(w.to(self.dev))

    # -- host views -------------------------------------------------------------

    def done(self) -> bool:
        return bool((self.gen_len >= self.max_new).all().item())

    def run(self, max_steps: int = 1_000_000) -> int:
        n = 0
        while n < max_steps and not self.done():
            self.step()
            n += 1
        return n

    def outputs(self) -> list[list[int]]:
        tok = self.tokens.cpu().numpy()
        lens = self.seq_len.cpu().numpy()
        return [tok[b, self.prompt_lens[b]: lens[b]].tolist() for b in range(self.B)]

    def outcome_rows(self, steps: int | None = None) -> np.ndarray:
        h = self.history.cpu().numpy()
        return h[: steps] if steps is not None else h
