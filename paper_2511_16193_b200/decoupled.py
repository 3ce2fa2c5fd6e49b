"""Decoupled speculation: drafting and verification on different GPUs,
pipeline depth 2 (paper §3/§4.1; reference ``sim.py:860-917``, ``1051-1092``).

Round r, per request:

* the verifier checks the window it received at the end of round r-1;
* meanwhile the drafter drafts the *next* window: the successor of the
  in-flight window (assuming it fully accepts) or, if none is in flight, a
  fresh window from the committed position;
* at the end of the round the drafter streams its windows (drafts [B, k],
  sizes [B]) to the verifier and the verifier streams its decisions
  (accepted, committed count, committed tokens [B, k+1]) back -- ~20 KB per
  round over NVLink (``NcclChannel``: batched NCCL P2P between ranks;
  ``run_local`` drives both roles in one process for single-GPU tests);
* a successor survives only if its predecessor fully accepted; otherwise it
  is charged as waste (``depth2_waste``, ``sim.py:1074-1080``) and the
  request's next round is a draft-only gap round.

Exact-match semantics make the committed tokens identical to plain decoding;
with the reference-acceptance drafter the per-request outcome stream
(proposed, accepted, committed, wasted) equals the reference simulator's
decoupled policy.  Bonus tokens are off (the successor starts at start + n).

Drafters on the drafter side: the reference-acceptance drafter, the n-gram
drafter (K4), and a small model (K5, ``ModelDrafter``) with its own paged KV
cache whose context is the committed tokens plus the in-flight window; a
rejected window pulls its cached length back to the corrected token.
"""

from __future__ import annotations

import math
import time

import numpy as np
import torch

from . import _native
from .engine import ModelDrafter, NgramDrafter, SyntheticDrafter, prefill_model
from .errors import ConfigError
from .model import DeviceModel


class NcclChannel:
    """torch.distributed P2P (NCCL over NVLink) between the drafter rank and
    the verifier rank: one batched isend/irecv per round."""

    def __init__(self, dist, peer: int):
        self.dist, self.peer = dist, peer

    def exchange(self, send: list, recv: list) -> None:
        ops = [self.dist.P2POp(self.dist.isend, t, self.peer) for t in send]
        ops += [self.dist.P2POp(self.dist.irecv, t, self.peer) for t in recv]
        for w in self.dist.batch_isend_irecv(ops):
            w.wait()


class HostChannel:
    """The same exchange staged through host memory over a CPU process
    group (gloo): lets the multi-process protocol run with several ranks on
    ONE GPU (tests), where NCCL refuses duplicate devices.  Not a product
    transport."""

    def __init__(self, dist, peer: int):
        self.dist, self.peer = dist, peer

    def exchange(self, send: list, recv: list) -> None:
        torch.cuda.synchronize()
        reqs = [self.dist.isend(t.cpu(), self.peer) for t in send]
        bufs = [torch.empty(t.shape, dtype=t.dtype) for t in recv]
        reqs += [self.dist.irecv(b, self.peer) for b in bufs]
        for r in reqs:
            r.wait()
        for t, b in zip(recv, bufs):
            t.copy_(b)


def _graph(fn):
    """Capture ``fn`` (static-shape device work, no host syncs) into a CUDA
    graph; returns the graph (replay() reruns ``fn`` on the same buffers)."""
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin()
        fn()
        g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    return g


class DraftSide:
    """Drafter GPU state: committed-token mirror + the in-flight window.

    Per round: :meth:`draft` fills ``out_drafts`` / ``out_nd`` (sent to the
    verifier), :meth:`apply` folds the verifier's decisions received into
    ``in_verified`` / ``in_accepted`` / ``in_committed`` / ``in_ctoks``.  Both
    are static-buffer device work, replayed from CUDA graphs after the first
    round (``graphs=True``)."""

    def __init__(self, prompts, max_new, k: int, drafter, device="cuda", graphs: bool = True, vocab: int = 0):
        if isinstance(drafter, (SyntheticDrafter, NgramDrafter, ModelDrafter)):
            self.drafter = drafter
            # wrong-token id space of the synthetic drafter
            self.vocab = (drafter.vocab or vocab) if isinstance(drafter, SyntheticDrafter) else vocab
        else:
            raise ConfigError("decoupled mode supports the n-gram, small-model and reference-acceptance drafters")
        self.lib = _native.lib()
        self.dev = torch.device(device)
        self.B, self.k = len(prompts), k
        lens = [len(p) for p in prompts]
        self.stride = int(math.ceil((max(l + n for l, n in zip(lens, max_new)) + 2 * k + 2) / 16) * 16)
        tok = np.zeros((self.B, self.stride), np.int32)
        for i, p in enumerate(prompts):
            tok[i, : len(p)] = p
        d = self.dev
        B = self.B
        self.tokens = torch.from_numpy(tok).to(d)
        self.seq_len = torch.tensor(lens, dtype=torch.int32, device=d)
        self.gen_len = torch.zeros(B, dtype=torch.int32, device=d)
        self.max_new = torch.tensor(max_new, dtype=torch.int32, device=d)
        self.inflight = torch.zeros(B, dtype=torch.int32, device=d)   # drafted tokens in flight
        self.drafts = torch.full((B, k), -1, dtype=torch.int32, device=d)
        self.nd = torch.zeros(B, dtype=torch.int32, device=d)
        self.g0 = torch.zeros(B, dtype=torch.int32, device=d)
        self.ctx = torch.zeros(B, dtype=torch.int32, device=d)
        self.scratch = torch.zeros(2 * B, dtype=torch.int64, device=d)
        # round I/O (static: graph-replayable, NCCL-sendable)
        self.out_drafts = torch.full((B, k), -1, dtype=torch.int32, device=d)
        self.out_nd = torch.zeros(B, dtype=torch.int32, device=d)
        self.in_verified = torch.zeros(B, dtype=torch.int32, device=d)
        self.in_accepted = torch.zeros(B, dtype=torch.int32, device=d)
        self.in_committed = torch.zeros(B, dtype=torch.int32, device=d)
        self.in_ctoks = torch.zeros((B, k + 1), dtype=torch.int32, device=d)
        self.use_graphs = graphs
        self._g_draft = self._g_apply = None
        if isinstance(drafter, ModelDrafter):
            self._attach_model(drafter, lens)

    def _attach_model(self, drafter, lens) -> None:
        """K5 on the drafter GPU: the small model's own paged KV cache over
        this side's token mirror.  Its context for window j+1 is the committed
        tokens plus in-flight window j; when window j is rejected the cached
        length is pulled back to the corrected token, whose KV (and all after
        it) the next catch-up recomputes (greedy drafting, T = 0)."""
        m, B, k, d = drafter.m, self.B, self.k, self.dev
        if m.max_tokens < B * (k + 2) or m.max_seqs < B or m.max_len < self.stride:
            raise ConfigError("drafter model capacity too small for the batch")
        self.dkv_len = torch.tensor([L - 1 for L in lens], dtype=torch.int32, device=d)
        self.m_token_ids = torch.zeros(B * (k + 2), dtype=torch.int32, device=d)
        self.m_positions = torch.zeros(B * (k + 2), dtype=torch.int32, device=d)
        self.m_seqs = torch.zeros((B, 8), dtype=torch.int32, device=d)
        self.m_logit_rows = torch.zeros(B, dtype=torch.int32, device=d)
        self.m_out = torch.zeros(B, dtype=torch.int32, device=d)
        self.max_key = self.stride - 1
        prefill_model(m, self.tokens, [L - 1 for L in lens])

    def _draft_model(self, st) -> None:
        m, lib = self.drafter.m, self.lib
        for step in range(self.k + 1):
            _native.check(lib.sr_draft_model_batch(
                self.B, self.k, step, self.tokens.data_ptr(), self.stride, self.ctx.data_ptr(),
                self.g0.data_ptr(), self.max_new.data_ptr(), self.dkv_len.data_ptr(), self.m_out.data_ptr(),
                self.drafts.data_ptr(), self.nd.data_ptr(), self.m_token_ids.data_ptr(),
                self.m_positions.data_ptr(), self.m_seqs.data_ptr(), self.m_logit_rows.data_ptr(), None, st),
                "sr_draft_model_batch")
            if step == 0:
                m.forward(self.m_token_ids, self.m_positions, self.m_seqs, num_seqs=self.B,
                          max_q_len=self.k + 2, max_key=self.max_key, out=self.m_out,
                          logit_rows=self.m_logit_rows)
            elif step < self.k:   # decode steps: one row per request, rows [0, B)
                m.forward(self.m_token_ids[:self.B], self.m_positions[:self.B], self.m_seqs, num_seqs=self.B,
                          max_q_len=1, max_key=self.max_key, out=self.m_out)

    def _draft(self) -> None:
        st, lib = _native.stream_handle(), self.lib
        _native.check(lib.sr_decoupled_draft_prep(self.B, self.seq_len.data_ptr(), self.gen_len.data_ptr(),
                                                  self.inflight.data_ptr(), self.g0.data_ptr(), self.ctx.data_ptr(),
                                                  st), "sr_decoupled_draft_prep")
        if isinstance(self.drafter, SyntheticDrafter):
            d = self.drafter
            _native.check(lib.sr_synthetic_draft(
                self.B, self.k, d.truth.data_ptr(), d.stride, self.max_new.data_ptr(), d.uniforms.data_ptr(),
                d.stride, d.p.data_ptr(), self.g0.data_ptr(), self.vocab, self.drafts.data_ptr(),
                self.nd.data_ptr(), st), "sr_synthetic_draft")
        elif isinstance(self.drafter, ModelDrafter):
            self._draft_model(st)
        else:
            d = self.drafter
            _native.check(lib.sr_ngram_propose(
                self.B, self.tokens.data_ptr(), self.stride, self.ctx.data_ptr(), d.min_n, d.max_n, self.k,
                self.drafts.data_ptr(), self.nd.data_ptr(), self.scratch.data_ptr(), st), "sr_ngram_propose")
        # cap at the budget, append behind the in-flight window, stage for the verifier
        _native.check(lib.sr_decoupled_draft_post(
            self.B, self.k, self.stride, self.max_new.data_ptr(), self.g0.data_ptr(), self.ctx.data_ptr(),
            self.drafts.data_ptr(), self.nd.data_ptr(), self.tokens.data_ptr(), self.out_drafts.data_ptr(),
            self.out_nd.data_ptr(), st), "sr_decoupled_draft_post")

    def _apply(self) -> None:
        dkv = self.dkv_len.data_ptr() if isinstance(self.drafter, ModelDrafter) else None
        _native.check(self.lib.sr_decoupled_draft_apply(
            self.B, self.k, self.stride, self.in_verified.data_ptr(), self.in_accepted.data_ptr(),
            self.in_committed.data_ptr(), self.in_ctoks.data_ptr(), self.out_nd.data_ptr(), self.inflight.data_ptr(),
            self.tokens.data_ptr(), self.seq_len.data_ptr(), self.gen_len.data_ptr(), dkv, _native.stream_handle()),
            "sr_decoupled_draft_apply")

    def draft(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Next window of every request: successor of the in-flight one, or
        fresh.  Returns (drafts [B, k], nd [B]); nd = 0 is an empty window
        (nothing proposed: verifying it commits the target's next token)."""
        if not self.use_graphs:
            self._draft()
        elif self._g_draft is None:
            self._draft()
            self._g_draft = _graph(self._draft)
        else:
            self._g_draft.replay()
        return self.out_drafts, self.out_nd

    def apply(self) -> None:
        """Fold the verifier's decisions (``in_*``) for the windows that were in flight."""
        if not self.use_graphs:
            self._apply()
        elif self._g_apply is None:
            self._apply()
            self._g_apply = _graph(self._apply)
        else:
            self._g_apply.replay()



class VerifySide:
    """Verifier GPU: the target model, the authoritative token buffer, and the
    windows received from the drafter (``in_drafts`` / ``in_nd``).

    Per round: :meth:`verify` checks the pending windows and fills the
    decision buffers ``out_verified`` / ``out_accepted`` / ``out_committed``
    / ``out_ctoks`` (sent to the drafter) and ``rows`` (outcome rows);
    :meth:`receive` installs the next windows.  Both replay CUDA graphs."""

    def __init__(self, model: DeviceModel, prompts, max_new, k: int, graphs: bool = True):
        from .engine import RolloutEngine

        self.eng = RolloutEngine(model, prompts, max_new, k=k, drafters=(NgramDrafter(),), bonus_token=False,
                                 history=1)
        self.k, self.B = k, len(prompts)
        d = self.eng.dev
        B = self.B
        # pending windows = the engine's drafter-0 draft slots (no copies)
        self.pending = self.eng.drafts[0]
        self.pending_nd = self.eng.ndraft[0]
        self.pending.fill_(-1)
        self.pending_nd.fill_(-1)                                   # -1: no window
        self.seq_before = torch.zeros(B, dtype=torch.int32, device=d)
        self.out_verified = torch.zeros(B, dtype=torch.int32, device=d)
        self.out_accepted = torch.zeros(B, dtype=torch.int32, device=d)
        self.out_committed = torch.zeros(B, dtype=torch.int32, device=d)
        self.out_ctoks = torch.zeros((B, k + 1), dtype=torch.int32, device=d)
        self.rows = torch.zeros((B, 4), dtype=torch.int32, device=d)
        self.in_drafts = torch.full((B, k), -1, dtype=torch.int32, device=d)
        self.in_nd = torch.zeros(B, dtype=torch.int32, device=d)
        self.use_graphs = graphs
        self._g_verify = self._g_receive = None

    def prefill(self):
        self.eng.prefill()

    def _verify(self) -> None:
        e = self.eng
        lib, st = e.lib, _native.stream_handle()
        self.seq_before.copy_(e.seq_len)
        # the pending windows live in the engine's drafter-0 slots (receive writes them there)
        _native.check(lib.sr_build_verify_batch(
            e.B, 1, e.k, e.tokens.data_ptr(), e.stride, e.seq_len.data_ptr(), e.gen_len.data_ptr(),
            e.max_new.data_ptr(), e.max_new_cap.data_ptr(), e.drafts.data_ptr(), e.ndraft.data_ptr(), None, None,
            e.token_ids.data_ptr(), e.positions.data_ptr(), e.seqs.data_ptr(), e.live_rows.data_ptr(), st),
            "sr_build_verify_batch")
        e.m.forward(e.token_ids, e.positions, e.seqs, num_seqs=e.B, max_q_len=e.k + 1, max_key=e.max_key,
                    out=e.target_ids, live_rows=e.live_rows)
        out = e.history[0]
        _native.check(lib.sr_accept_commit(
            e.m.handle, e.B, 1, e.seqs.data_ptr(), e.token_ids.data_ptr(), e.target_ids.data_ptr(), e.tokens.data_ptr(),
            e.stride, e.seq_len.data_ptr(), e.gen_len.data_ptr(), e.max_new.data_ptr(), 0, out.data_ptr(),
            e.bon.data_ptr(), st), "sr_accept_commit")
        _native.check(lib.sr_decoupled_verify_post(
            e.B, e.k, e.stride, out.data_ptr(), e.bon.data_ptr(), e.tokens.data_ptr(), self.seq_before.data_ptr(),
            self.rows.data_ptr(), self.out_verified.data_ptr(), self.out_accepted.data_ptr(),
            self.out_committed.data_ptr(), self.out_ctoks.data_ptr(), st), "sr_decoupled_verify_post")

    def _receive(self) -> None:
        e = self.eng
        _native.check(e.lib.sr_decoupled_verify_receive(
            self.B, self.k, self.out_verified.data_ptr(), self.out_accepted.data_ptr(), self.out_committed.data_ptr(),
            self.in_drafts.data_ptr(), self.in_nd.data_ptr(), self.rows.data_ptr(), self.pending.data_ptr(),
            self.pending_nd.data_ptr(), _native.stream_handle()), "sr_decoupled_verify_receive")

    def verify(self) -> None:
        """Verify the pending windows into the ``out_*`` buffers and ``rows``."""
        if not self.use_graphs:
            self._verify()
        elif self._g_verify is None:
            self._verify()
            self._g_verify = _graph(self._verify)
        else:
            self._g_verify.replay()

    def receive(self) -> torch.Tensor:
        """Install the drafter's windows (``in_*``); successors of rejected
        windows are dropped and charged to the rejected outcome (depth-2
        waste).  Returns the round's outcome rows (device, [B, 4])."""
        if not self.use_graphs:
            self._receive()
        elif self._g_receive is None:
            self._receive()
            self._g_receive = _graph(self._receive)
        else:
            self._g_receive.replay()
        return self.rows

    def done(self) -> bool:
        return self.eng.done()


def run_local(model: DeviceModel, prompts, max_new, k: int, drafter, max_rounds: int = 100000,
              graphs: bool = True):
    """Both roles on one GPU (tests): returns (outputs, outcome rows per round)."""
    D = DraftSide(prompts, max_new, k, drafter, device=model.dev, graphs=graphs, vocab=model.s.vocab)
    V = VerifySide(model, prompts, max_new, k, graphs=graphs)
    V.prefill()
    history = []
    # round 0: draft-only (nothing in flight yet); the verifier's decision
    # buffers start as "nothing verified"
    drafts, nd = D.draft()
    V.in_drafts.copy_(drafts)
    V.in_nd.copy_(nd)
    V.receive()
    D.apply()
    for _ in range(max_rounds):
        if V.done():
            break
        V.verify()
        drafts, nd = D.draft()                    # concurrent with verify on two GPUs
        V.in_drafts.copy_(drafts)
        V.in_nd.copy_(nd)
        for dst, src in ((D.in_verified, V.out_verified), (D.in_accepted, V.out_accepted),
                         (D.in_committed, V.out_committed), (D.in_ctoks, V.out_ctoks)):
            dst.copy_(src)
        rows = V.receive()
        D.apply()
        history.append(rows.clone())
    h = torch.stack(history).cpu().numpy() if history else np.zeros((0, D.B, 4), np.int32)
    return V.eng.outputs(), h


def pairing(world: int, drafters: int) -> dict:
    """Ranks [0, drafters) draft, the rest verify; verifier v is served by
    drafter (v - drafters) % drafters (configs[3]: 2 draft + 6 verify)."""
    if not (1 <= drafters < world):
        raise ConfigError("need at least one drafter and one verifier rank")
    return {v: (v - drafters) % drafters for v in range(drafters, world)}


def run_ranks(dist, rank: int, world: int, drafters: int, shards: dict, k: int, make_drafter,
              make_model=None, max_rounds: int = 1_000_000, graphs: bool = True, round_times=None,
              channel=NcclChannel):
    """Decoupled rollout across ranks (one process per GPU).

    ``shards[v]`` = (prompts, max_new) of verifier rank v.  Drafter ranks run
    one :class:`DraftSide` per verifier they serve; verifier ranks run a
    :class:`VerifySide` on ``make_model()``.  Each round is one batched NCCL
    isend/irecv per (drafter, verifier) pair on static buffers; each side's
    per-round device work replays a CUDA graph.  Returns (outputs, outcome
    rows, rounds) on verifier ranks, (None, None, rounds) on drafter ranks.
    ``round_times`` (a list, verifier ranks): host time after each round's
    exchange completed (the round's device work is done then).
    ``channel``: :class:`NcclChannel` (device buffers over NVLink) or
    :class:`HostChannel` (tests: several ranks sharing one GPU).
    """
    dev = torch.device("cuda", torch.cuda.current_device())
    pairs = pairing(world, drafters)
    if rank < drafters:
        mine = [v for v, d in pairs.items() if d == rank]
        sides, done = {}, {}
        for v in mine:
            prompts, max_new = shards[v]
            drafter = make_drafter(v)
            sides[v] = DraftSide(prompts, max_new, k, drafter, device=dev, graphs=graphs)
            done[v] = torch.zeros(1, dtype=torch.int32, device=dev)
        live = set(mine)
        rounds = 0
        while live and rounds < max_rounds:
            for v in sorted(live):
                D = sides[v]
                drafts, nd = D.draft()
                channel(dist, v).exchange(
                    [drafts, nd], [D.in_verified, D.in_accepted, D.in_committed, D.in_ctoks, done[v]])
                D.apply()
                if int(done[v].item()):
                    live.discard(v)
            rounds += 1
        return None, None, rounds
    prompts, max_new = shards[rank]
    V = VerifySide(make_model(), prompts, max_new, k, graphs=graphs)
    V.prefill()
    peer = pairs[rank]
    done = torch.zeros(1, dtype=torch.int32, device=dev)
    history, rounds = [], 0
    ev = []
    while rounds < max_rounds:
        if round_times is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        V.verify()
        if round_times is not None:
            e1.record()
            ev.append((e0, e1))
        done.fill_(1 if V.done() else 0)
        channel(dist, peer).exchange(
            [V.out_verified, V.out_accepted, V.out_committed, V.out_ctoks, done], [V.in_drafts, V.in_nd])
        rows = V.receive()
        if rounds > 0:
            history.append(rows.clone())
        rounds += 1
        finished = int(done.item())
        if round_times is not None:
            round_times.append(time.perf_counter())
        if finished:
            break
    h = torch.stack(history).cpu().numpy() if history else None
    if round_times is not None:
        torch.cuda.synchronize()
        round_times.append([a.elapsed_time(b) for a, b in ev])   # last entry: verify ms per round
    return V.eng.outputs(), h, rounds
