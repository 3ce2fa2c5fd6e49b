"""SpecActor's rollout policies driving the real engine (SURVEY §8a a10/a11,
§8f.2): the per-request acceptance estimators fed from device outcome rows,
Best-of-N drafters assigned to the tail when the batch drains, and
request-level window reconfiguration -- on ``RolloutEngine`` steps instead of
the reference's virtual-time executors.

Mapping of the reference's mechanisms (``sim.py``) onto one engine:

* Workers and drain.  The reference frees a worker (GPU group) when its
  executor drains and hands it to ``bon.assign_bon`` (``sim.py:373-392``,
  ``bon.py:79-139``).  Here the batch is one engine; every ``b_max``
  requests that finish free ``b_max * (k + 1)`` verify rows -- one "worker"
  with room for ``b_max`` extra drafter windows -- and ``assign_bon`` places
  it on the least-staffed method and packs the slowest live requests onto
  it.  An assignment turns drafter n of request b on (``set_active``); its
  window is verified in the same forward as the incumbent's and the longest
  accepted prefix wins (K3), so no replica start-up cost exists.
* Estimators.  Every step's outcome rows come back with the host-facing
  step (``capture_io``); drafter n of request b records (proposed, accepted)
  into a K-outcome ring with the reference estimator's semantics
  (``workload.py:42-56``: accepted / proposed over the last K outcomes, the
  prior until a proposal was seen), vectorized over the batch.
* Reconfiguration.  Every ``reconfig_interval`` committed tokens once the
  batch is in its tail, ``planner.reconfigure`` (Alg. 2, ``sim.py:445-510``)
  picks a window for the slower half of the live requests from their
  estimates; ``set_windows`` caps them on device (mixed windows in one
  forward).

Exactness is untouched: every policy only changes which drafts are
verified, and verification is exact match against the target, so the
committed tokens equal plain decoding's.  The driver logs the reference's
event schema (``sim.py:363-369``) with CUDA-event timestamps.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .bon import ClusterState, assign_bon, release_pair
from .errors import ConfigError
from .workload import AcceptanceEstimator, Request


@dataclass
class Event:
    """One entry of the reference's event log (``sim.py:363-369``)."""

    time_ms: float
    kind: str
    worker: str
    request: int
    payload: dict = field(default_factory=dict)

    def as_dict(self) -> dict:
        return {"time_ms": round(self.time_ms, 3), "kind": self.kind, "worker": self.worker,
                "request": self.request, "payload": self.payload}


@dataclass
class RolloutReport:
    makespan_ms: float            # device time: first step launch -> the last committing step done
    steps: int
    committed: int
    windows: int                  # verified (request, drafter) windows
    proposed: int
    accepted: int
    bon_pairs: int                # (request, method) drafters turned on
    reconfigs: int
    finish_ms: dict               # request id -> finish time (ms)
    live_rows: list               # verify rows per step (= the compacted batch's rows)
    events: list

    @property
    def tokens_per_s(self) -> float:
        return self.committed / (self.makespan_ms * 1e-3) if self.makespan_ms > 0 else 0.0


class OutcomeRings:
    """Per-(request, drafter) acceptance estimators over the last ``window``
    outcomes, batched: the reference's ``AcceptanceEstimator`` semantics on
    numpy rings."""

    def __init__(self, B: int, N: int, window: int, priors):
        self.p = np.zeros((B, N, window), np.int64)
        self.a = np.zeros((B, N, window), np.int64)
        self.count = np.zeros((B, N), np.int64)
        self.window = window
        self.prior = np.asarray(priors, np.float64).reshape(1, N).repeat(B, 0)

    def record(self, mask: np.ndarray, proposed: np.ndarray, accepted: np.ndarray) -> None:
        """Append (proposed, accepted)[b, n] where mask[b, n]."""
        b, n = np.nonzero(mask)
        slot = self.count[b, n] % self.window
        self.p[b, n, slot] = proposed[b, n]
        self.a[b, n, slot] = accepted[b, n]
        self.count[b, n] += 1

    def reset(self, b: int) -> None:
        """Slot b took a new request: back to the priors."""
        self.p[b] = 0
        self.a[b] = 0
        self.count[b] = 0

    def estimate(self) -> np.ndarray:
        tp, ta = self.p.sum(-1), self.a.sum(-1)
        return np.where(tp > 0, ta / np.maximum(tp, 1), self.prior)

    def estimator(self, b: int, n: int) -> AcceptanceEstimator:
        """The reference object for (b, n), ring in recording order."""
        est = AcceptanceEstimator(self.window, float(self.prior[b, n]))
        c = int(self.count[b, n])
        for i in range(max(0, c - self.window), c):
            est.record(int(self.p[b, n, i % self.window]), int(self.a[b, n, i % self.window]))
        return est


@dataclass(frozen=True)
class Placement:
    """The plan search's answer for a batch (reference ``planner.py:113-211``,
    reported side by side by the CLI's ``plan`` command ``cli.py:406-460``):
    the mode with the higher modeled throughput, its window, and both plans."""

    mode: str            # "coupled" | "decoupled"
    window: int
    tgs_estimate: float
    decoupled: object    # planner.ExecutionPlan
    coupled: object      # planner.CoupledPlan


def choose_placement(batch: int, model, p: float, method: str | None = None) -> Placement:
    """Run both plan searches on a (measured) cost model and pick the mode
    with the higher tokens/GPU/s estimate; ties go to coupled (no drafter
    GPUs to dedicate)."""
    from .planner import search_plan, search_plan_coupled

    dec = search_plan(batch, model, p, method)
    cpl = search_plan_coupled(batch, model, p, method)
    if dec.tgs_estimate > cpl.tgs_estimate:
        return Placement("decoupled", dec.window, dec.tgs_estimate, dec, cpl)
    return Placement("coupled", cpl.window, cpl.tgs_estimate, dec, cpl)


class RolloutDriver:
    """Runs a :class:`~paper_2511_16193_b200.engine.RolloutEngine` to
    completion through its host-facing step with SpecActor's tail policies.

    ``requests[b]`` is the reference ``Request`` of slot b (ids, latent
    acceptance); ``methods[n]`` names drafter n (drafter 0 is the incumbent,
    always on).  ``bon_on_drain``: extra drafters start off and are assigned
    by ``assign_bon`` as the batch drains.  ``reconfig``: (plan, cost model)
    for ``planner.reconfigure``, or None.
    """

    def __init__(self, eng, requests: list[Request], methods: list[str], *, bon_on_drain: bool = True,
                 b_max: int = 8, bon_policy: str = "greedy", reconfig=None, reconfig_interval: int = 1000,
                 tail_fraction: float = 0.5, estimator_window: int = 64, priors: dict | None = None,
                 log_events: bool = False, straggler=None, placement: Placement | None = None):
        if len(requests) != eng.B or len(methods) != eng.N:
            raise ConfigError("one request per slot and one method name per drafter")
        self.eng, self.reqs, self.methods = eng, list(requests), list(methods)
        self.bon_on_drain = bon_on_drain and eng.N > 1
        self.b_max, self.bon_policy = b_max, bon_policy
        self.reconfig, self.reconfig_interval = reconfig, reconfig_interval
        self.tail_fraction = tail_fraction
        priors = priors or {}
        self.rings = OutcomeRings(eng.B, eng.N, estimator_window, [priors.get(m, 0.5) for m in methods])
        self.log_events = log_events
        self.state = ClusterState(b_max=b_max)
        self.pairs: dict[tuple[int, str], str] = {}   # live (request id, method) -> worker
        # cross-rank straggler pulls (straggler.StragglerPull), run at
        # quiescent points: every `interval` steps, and continuously once
        # this rank has drained (it is then a pull target)
        self.straggler = straggler
        # the plan search's window reaches the engine (a decoupled placement
        # runs through decoupled.run_ranks, not a single-engine driver)
        self.placement = placement
        if placement is not None:
            if placement.mode != "coupled":
                raise ConfigError("decoupled placement: run it with decoupled.run_ranks "
                                  f"(g_d = {placement.decoupled.g_d} drafter GPUs per group)")
            eng.set_windows(np.full(eng.B, max(1, min(eng.k, placement.window)), np.int32))
        self._gen = self._budget = self._budget_h = None
        self.released: set[int] = set()          # slots whose request moved to another rank
        self.stashed: dict[int, list[int]] = {}  # outputs of finished requests whose slot was reused

    # -- slot movement (straggler pulls) --------------------------------------------

    def slot_states(self):
        """(live [(slot, request id, incumbent estimate)], free slots)."""
        est = self.rings.estimate()[:, 0]   # the incumbent's ring estimates, vectorised
        live, free = [], []
        for b in range(self.eng.B):
            if self._gen[b] < self._budget[b]:
                live.append((b, self.reqs[b].id, float(est[b])))
            else:
                free.append(b)
        return live, free

    def release_slot(self, b: int) -> None:
        """Slot b's request leaves this rank: stop it here for good (the
        pinned host budget is what every captured step copies to the device)
        and hand back its Best-of-N drafters."""
        self._budget[b] = self._gen[b]
        self._budget_h[b] = int(self._gen[b])
        self.released.add(b)
        rid = self.reqs[b].id
        for method in self.methods[1:]:
            w = self.pairs.pop((rid, method), None)
            if w is not None:
                release_pair(self.state, rid, method, w)
        if self.eng.N > 1:
            mask = self.eng.active.cpu().numpy()
            mask[1:, b] = 0
            self.eng.set_active(mask)

    def stash_slot(self, b: int) -> None:
        """Keep the output of slot b's finished request before the slot is
        reused by an adopted one."""
        if b not in self.released:
            self.stashed[self.reqs[b].id] = self.eng.outputs()[b]

    def outputs_by_id(self) -> dict[int, list[int]]:
        """Every request that finished on this engine: request id -> tokens."""
        out = dict(self.stashed)
        for b, toks in enumerate(self.eng.outputs()):
            if b not in self.released:
                out[self.reqs[b].id] = toks
        return out

    def adopt_slot(self, b: int, request: Request) -> None:
        """Slot b now holds ``request`` (already installed on the device by
        ``migrate.recv_requests``): host lengths, budget and a fresh
        estimator follow it."""
        self.reqs[b] = request
        self.released.discard(b)
        self._gen[b] = int(self.eng.gen_len[b])
        self._budget[b] = int(self.eng.max_new[b])
        self._budget_h[b] = int(self._budget[b])
        self.rings.reset(b)
        if self.eng.N > 1:
            mask = self.eng.active.cpu().numpy()
            mask[1:, b] = 0
            self.eng.set_active(mask)

    def log_event(self, events: list, t_ms: float, kind: str, worker: str, rid: int, detail: dict) -> None:
        if self.log_events:
            events.append(Event(t_ms, kind, worker, rid, detail))

    # -- policies ------------------------------------------------------------------

    def _live_requests(self, live: np.ndarray) -> list[Request]:
        """Reference Request views of the live slots with their incumbent
        estimators (assign_bon ranks slowest first)."""
        out = []
        for b in np.nonzero(live)[0]:
            r = self.reqs[b]
            out.append(Request(id=r.id, prompt_len=r.prompt_len, true_len=r.true_len,
                               latent_accept=r.latent_accept, rate_estimate=self.rings.estimator(int(b), 0)))
        return out

    def _drain(self, live: np.ndarray, freed: list[str], t_ms: float, events: list) -> int:
        if not freed:
            return 0
        slot_of = {r.id: b for b, r in enumerate(self.reqs)}
        extra = self.methods[1:]
        got = assign_bon(self._live_requests(live), extra, freed, self.state, self.bon_policy)
        mask = self.eng.active.cpu().numpy()
        for (rid, method), worker in got.pairs.items():
            mask[self.methods.index(method), slot_of[rid]] = 1
            self.pairs[(rid, method)] = worker
            if self.log_events:
                events.append(Event(t_ms, "bon_assign", worker, rid, {"method": method}))
        self.eng.set_active(mask)
        return len(got.pairs)

    def _reconfigure(self, live: np.ndarray, t_ms: float, events: list) -> int:
        from .planner import reconfigure

        plan, model = self.reconfig
        reqs = self._live_requests(live)
        if not reqs:
            return 0
        plans = reconfigure(plan, reqs, model)
        if not plans:
            return 0
        slot_of = {r.id: b for b, r in enumerate(self.reqs)}
        w = self.eng.window.cpu().numpy()
        for p in plans:
            w[slot_of[p.request_id]] = max(1, min(self.eng.k, p.window))
            if self.log_events:
                events.append(Event(t_ms, "reconfig", "engine", p.request_id, {"window": p.window, "mode": p.mode}))
        self.eng.set_windows(w)
        return len(plans)

    # -- the loop ------------------------------------------------------------------

    def run(self, max_steps: int = 1_000_000) -> RolloutReport:
        eng = self.eng
        B, N, k = eng.B, eng.N, eng.k
        if self.bon_on_drain:
            off = np.zeros((N, B), np.int32)
            eng.set_active(off)                                    # incumbents only
        budget = eng.max_new.cpu().numpy().astype(np.int32)
        gen = eng.gen_len.cpu().numpy().astype(np.int64)
        budget_h = torch.from_numpy(budget.copy()).pin_memory()
        self._gen, self._budget, self._budget_h = gen, budget, budget_h.numpy()
        cols = 4 * N + k + 2
        res = [torch.zeros((B, cols), dtype=torch.int32).pin_memory() for _ in range(2)]
        graphs = [eng.capture_io(budget_h, r) for r in res]
        done_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        start = torch.cuda.Event(enable_timing=True)
        events: list = []
        finish_ms: dict = {}
        live_rows: list = []
        windows = proposed = accepted = committed = bon_pairs = reconfigs = 0
        freed_pending = 0
        worker_seq = 0
        since_reconfig = 0
        torch.cuda.synchronize()
        start.record()
        step = 0
        last_ms = 0.0
        pending = None          # the launched step whose results are not read yet
        all_done = not (gen < budget).any()
        hook = self.straggler
        last_hook = 0
        while True:
            # a straggler exchange needs every step read: launch nothing this round
            due = hook is not None and (all_done or step >= max_steps or step - last_hook >= hook.interval)
            launched = None
            if not due and step < max_steps and not all_done:
                # launch step s, then read step s-1's results while s runs;
                # policy decisions made now apply from step s+1
                eng.step_io(graphs[step % 2])
                done_ev[step % 2].record()
                launched = step
                step += 1
            if pending is not None:
                done_ev[pending % 2].synchronize()
                t_ms = start.elapsed_time(done_ev[pending % 2])
                r = res[pending % 2].numpy()
                live = gen < budget
                rows = r[:, : 4 * N].reshape(B, N, 4)
                active_w = (rows[:, :, 0] + rows[:, :, 2]) > 0        # verified windows
                if active_w.any():
                    last_ms = t_ms
                    live_rows.append(int(rows[active_w][:, 0].sum() + active_w.sum()))
                self.rings.record(active_w, rows[:, :, 0], rows[:, :, 1])
                c = rows[:, :, 2].sum(1)
                gen += c
                step_committed = int(c.sum())
                committed += step_committed
                since_reconfig += step_committed
                windows += int(active_w.sum())
                proposed += int(rows[:, :, 0][active_w].sum())
                accepted += int(rows[:, :, 1][active_w].sum())
                if self.log_events:
                    for b in np.nonzero(active_w.any(1))[0]:
                        rid = self.reqs[b].id
                        win = int(np.argmax(rows[b, :, 2] > 0))
                        events.append(Event(t_ms, "verify", f"drafter-{win}", rid,
                                            {"proposed": int(rows[b, win, 0]), "accepted": int(rows[b, win, 1]),
                                             "drafters": int(active_w[b].sum())}))
                        events.append(Event(t_ms, "commit", "engine", rid, {"tokens": int(c[b])}))
                newly = live & (gen >= budget)
                for b in np.nonzero(newly)[0]:
                    rid = self.reqs[b].id
                    finish_ms[rid] = t_ms
                    if self.log_events:
                        events.append(Event(t_ms, "finish", "engine", rid, {}))
                    for method in self.methods[1:]:
                        w = self.pairs.pop((rid, method), None)
                        if w is not None:
                            release_pair(self.state, rid, method, w)
                freed_pending += int(newly.sum())
                still = gen < budget
                all_done = not still.any()
                if self.bon_on_drain and freed_pending >= self.b_max and not all_done:
                    freed = []
                    while freed_pending >= self.b_max:
                        freed.append(f"rows-{worker_seq}")
                        worker_seq += 1
                        freed_pending -= self.b_max
                    bon_pairs += self._drain(still, freed, t_ms, events)
                in_tail = still.sum() <= self.tail_fraction * B
                if self.reconfig is not None and in_tail and since_reconfig >= self.reconfig_interval:
                    since_reconfig = 0
                    reconfigs += self._reconfigure(still, t_ms, events)
            pending = launched
            if pending is not None:
                continue
            if hook is None:
                break
            last_hook = step
            t_ms = start.elapsed_time(done_ev[(step - 1) % 2]) if step else 0.0
            keep = hook(self, all_done or step >= max_steps, t_ms, events, can_run=step < max_steps)
            all_done = not (gen < budget).any()
            if not keep:
                break
        torch.cuda.synchronize()
        return RolloutReport(makespan_ms=last_ms, steps=step, committed=committed, windows=windows,
                             proposed=proposed, accepted=accepted, bon_pairs=bon_pairs, reconfigs=reconfigs,
                             finish_ms=finish_ms, live_rows=live_rows, events=[e.as_dict() for e in events])
