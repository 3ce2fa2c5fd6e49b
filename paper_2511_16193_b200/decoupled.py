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
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native
from .engine import NgramDrafter, SyntheticDrafter
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


class DraftSide:
    """Drafter GPU state: committed-token mirror + the in-flight window."""

    def __init__(self, prompts, max_new, k: int, drafter, device="cuda"):
        if isinstance(drafter, SyntheticDrafter) or isinstance(drafter, NgramDrafter):
            self.drafter = drafter
        else:
            raise ConfigError("decoupled mode supports the n-gram and reference-acceptance drafters")
        self.lib = _native.lib()
        self.dev = torch.device(device)
        self.B, self.k = len(prompts), k
        lens = [len(p) for p in prompts]
        self.stride = int(math.ceil((max(l + n for l, n in zip(lens, max_new)) + 2 * k + 2) / 16) * 16)
        tok = np.zeros((self.B, self.stride), np.int32)
        for i, p in enumerate(prompts):
            tok[i, : len(p)] = p
        d = self.dev
        self.tokens = torch.from_numpy(tok).to(d)
        self.seq_len = torch.tensor(lens, dtype=torch.int32, device=d)
        self.gen_len = torch.zeros(self.B, dtype=torch.int32, device=d)
        self.max_new = torch.tensor(max_new, dtype=torch.int32, device=d)
        self.inflight = torch.zeros(self.B, dtype=torch.int32, device=d)   # drafted tokens in flight
        self.drafts = torch.full((self.B, k), -1, dtype=torch.int32, device=d)
        self.nd = torch.zeros(self.B, dtype=torch.int32, device=d)
        self.scratch = torch.zeros(2 * self.B, dtype=torch.int64, device=d)
        self.ar = torch.arange(k, device=d)

    def draft(self) -> tuple[torch.Tensor, torch.Tensor]:
        """Next window of every request: successor of the in-flight one, or
        fresh.  Returns (drafts [B, k], nd [B]); nd = 0 means no window."""
        st = _native.stream_handle()
        g0 = self.gen_len + self.inflight                       # first drafted output position
        ctx = self.seq_len + self.inflight                      # context incl. in-flight drafts
        room = (self.max_new - g0).clamp(min=0)
        if isinstance(self.drafter, SyntheticDrafter):
            d = self.drafter
            _native.check(self.lib.sr_synthetic_draft(
                self.B, self.k, d.truth.data_ptr(), d.stride, self.max_new.data_ptr(), d.uniforms.data_ptr(),
                d.stride, d.p.data_ptr(), g0.contiguous().data_ptr(), self._vocab, self.drafts.data_ptr(),
                self.nd.data_ptr(), st), "sr_synthetic_draft")
        else:
            d = self.drafter
            _native.check(self.lib.sr_ngram_propose(
                self.B, self.tokens.data_ptr(), self.stride, ctx.contiguous().data_ptr(), d.min_n, d.max_n, self.k,
                self.drafts.data_ptr(), self.nd.data_ptr(), self.scratch.data_ptr(), st), "sr_ngram_propose")
        self.nd = torch.minimum(self.nd, room.to(torch.int32))
        # append the new window after the in-flight one (context of the next successor)
        cols = (ctx[:, None] + self.ar[None, :]).clamp(max=self.stride - 1).long()
        keep = self.ar[None, :] < self.nd[:, None]
        self.tokens.scatter_(1, cols, torch.where(keep, self.drafts, self.tokens.gather(1, cols)))
        return self.drafts.clone(), self.nd.clone()

    def apply(self, sent_nd, verified, accepted, committed, ctoks) -> None:
        """Fold the verifier's decisions for the windows that were in flight."""
        full = verified & (accepted == self.inflight)
        part = verified & ~full
        # partial: accepted prefix + corrected token
        pos = (self.seq_len + accepted).clamp(max=self.stride - 1).long()
        corr = ctoks.gather(1, accepted.clamp(max=self.k).long()[:, None])[:, 0]
        self.tokens.scatter_(1, pos[:, None], torch.where(part, corr, self.tokens.gather(1, pos[:, None])[:, 0])[:, None])
        adv = torch.where(verified, committed, torch.zeros_like(committed))
        self.seq_len += adv
        self.gen_len += adv
        # in flight next round: the window just drafted, unless its predecessor was rejected
        survive = ~part
        self.inflight = torch.where(survive, sent_nd, torch.zeros_like(sent_nd))

    _vocab = 0


class VerifySide:
    """Verifier GPU: the target model, the authoritative token buffer, and the
    windows received from the drafter."""

    def __init__(self, model: DeviceModel, prompts, max_new, k: int):
        from .engine import RolloutEngine

        self.eng = RolloutEngine(model, prompts, max_new, k=k, drafters=(NgramDrafter(),), bonus_token=False,
                                 history=1)
        self.k, self.B = k, len(prompts)
        d = self.eng.dev
        self.pending = torch.full((self.B, k), -1, dtype=torch.int32, device=d)
        self.pending_nd = torch.full((self.B,), -1, dtype=torch.int32, device=d)  # -1: no window

    def prefill(self):
        self.eng.prefill()

    def verify(self):
        """Verify the pending windows; returns (verified mask, accepted,
        committed, committed tokens [B, k+1], outcome rows [B, 4])."""
        e = self.eng
        lib, st = e.lib, _native.stream_handle()
        e.drafts[0].copy_(self.pending)
        e.ndraft[0].copy_(self.pending_nd)
        seq_before = e.seq_len.clone()
        _native.check(lib.sr_build_verify_batch(
            e.B, 1, e.k, e.tokens.data_ptr(), e.stride, e.seq_len.data_ptr(), e.gen_len.data_ptr(),
            e.max_new.data_ptr(), e.drafts.data_ptr(), e.ndraft.data_ptr(), e.token_ids.data_ptr(),
            e.positions.data_ptr(), e.seqs.data_ptr(), st), "sr_build_verify_batch")
        e.m.forward(e.token_ids, e.positions, e.seqs, num_seqs=e.B, max_q_len=e.k + 1, max_key=e.max_key,
                    out=e.target_ids)
        out = e.history[0]
        _native.check(lib.sr_accept_commit(
            e.B, 1, e.seqs.data_ptr(), e.token_ids.data_ptr(), e.target_ids.data_ptr(), e.tokens.data_ptr(),
            e.stride, e.seq_len.data_ptr(), e.gen_len.data_ptr(), e.max_new.data_ptr(), 0, out.data_ptr(),
            e.bon.data_ptr(), st), "sr_accept_commit")
        rows = out.clone()
        verified = e.bon >= 0
        accepted, committed = rows[:, 1].clone(), rows[:, 2].clone()
        cols = (seq_before[:, None] + torch.arange(self.k + 1, device=e.dev)[None, :]).clamp(max=e.stride - 1)
        ctoks = e.tokens.gather(1, cols.long())
        return verified, accepted, committed, ctoks, rows

    def receive(self, drafts, nd, verified, accepted, rows):
        """Install the drafter's windows; successors of rejected windows are
        dropped and charged to the rejected outcome (depth-2 waste)."""
        full = verified & (accepted == rows[:, 0])
        part = verified & ~full
        ok = (~verified | full) & (nd > 0)
        self.pending.copy_(drafts)
        self.pending_nd.copy_(torch.where(ok, nd, torch.full_like(nd, -1)))
        rows[:, 3] += torch.where(part, nd, torch.zeros_like(nd))
        return rows

    def done(self) -> bool:
        return self.eng.done()


def run_local(model: DeviceModel, prompts, max_new, k: int, drafter, max_rounds: int = 100000):
    """Both roles on one GPU (tests): returns (outputs, outcome rows per round)."""
    if isinstance(drafter, SyntheticDrafter):
        DraftSide._vocab = drafter.vocab or model.s.vocab
    D = DraftSide(prompts, max_new, k, drafter, device=model.dev)
    V = VerifySide(model, prompts, max_new, k)
    V.prefill()
    history = []
    # round 0: draft-only (nothing in flight yet)
    drafts, nd = D.draft()
    V.receive(drafts, nd, torch.zeros(D.B, dtype=torch.bool, device=model.dev),
              torch.zeros_like(nd), torch.zeros((D.B, 4), dtype=torch.int32, device=model.dev))
    D.apply(nd, torch.zeros(D.B, dtype=torch.bool, device=model.dev), torch.zeros_like(nd),
            torch.zeros_like(nd), torch.zeros((D.B, k + 1), dtype=torch.int32, device=model.dev))
    for _ in range(max_rounds):
        if V.done():
            break
        verified, accepted, committed, ctoks, rows = V.verify()
        drafts, nd = D.draft()                    # concurrent with verify on two GPUs
        rows = V.receive(drafts, nd, verified, accepted, rows)
        D.apply(nd, verified, accepted, committed, ctoks)
        history.append(rows.cpu().numpy())
    return V.eng.outputs(), np.stack(history) if history else np.zeros((0, D.B, 4), np.int32)


def pairing(world: int, drafters: int) -> dict:
    """Ranks [0, drafters) draft, the rest verify; verifier v is served by
    drafter (v - drafters) % drafters (configs[3]: 2 draft + 6 verify)."""
    if not (1 <= drafters < world):
        raise ConfigError("need at least one drafter and one verifier rank")
    return {v: (v - drafters) % drafters for v in range(drafters, world)}


def run_ranks(dist, rank: int, world: int, drafters: int, shards: dict, k: int, make_drafter,
              make_model=None, max_rounds: int = 1_000_000):
    """Decoupled rollout across ranks (one process per GPU).

    ``shards[v]`` = (prompts, max_new) of verifier rank v.  Drafter ranks run
    one :class:`DraftSide` per verifier they serve; verifier ranks run a
    :class:`VerifySide` on ``make_model()``.  Each round is one batched NCCL
    isend/irecv per (drafter, verifier) pair.  Returns (outputs, outcome
    rows, rounds) on verifier ranks, (None, None, rounds) on drafter ranks.
    """
    dev = torch.device("cuda", torch.cuda.current_device())
    pairs = pairing(world, drafters)
    if rank < drafters:
        mine = [v for v, d in pairs.items() if d == rank]
        sides = {}
        for v in mine:
            prompts, max_new = shards[v]
            drafter = make_drafter(v)
            if isinstance(drafter, SyntheticDrafter):
                DraftSide._vocab = drafter.vocab
            sides[v] = DraftSide(prompts, max_new, k, drafter, device=dev)
        live = set(mine)
        rounds = 0
        while live and rounds < max_rounds:
            for v in sorted(live):
                D = sides[v]
                drafts, nd = D.draft()
                B = D.B
                dec = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(3)]
                ctoks = torch.empty((B, k + 1), dtype=torch.int32, device=dev)
                done = torch.empty(1, dtype=torch.int32, device=dev)
                NcclChannel(dist, v).exchange([drafts, nd], dec + [ctoks, done])
                D.apply(nd, dec[0] > 0, dec[1], dec[2], ctoks)
                if int(done.item()):
                    live.discard(v)
            rounds += 1
        return None, None, rounds
    prompts, max_new = shards[rank]
    V = VerifySide(make_model(), prompts, max_new, k)
    V.prefill()
    peer = pairs[rank]
    history, rounds = [], 0
    while rounds < max_rounds:
        verified, accepted, committed, ctoks, rows = V.verify()
        done = torch.tensor([1 if V.done() else 0], dtype=torch.int32, device=dev)
        drafts = torch.empty((V.B, k), dtype=torch.int32, device=dev)
        nd = torch.empty(V.B, dtype=torch.int32, device=dev)
        NcclChannel(dist, peer).exchange([verified.to(torch.int32), accepted, committed, ctoks, done],
                                         [drafts, nd])
        rows = V.receive(drafts, nd, verified, accepted, rows)
        if rounds > 0:
            history.append(rows.cpu().numpy())
        rounds += 1
        if int(done.item()):
            break
    return V.eng.outputs(), np.stack(history) if history else None, rounds
