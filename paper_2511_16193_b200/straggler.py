"""Straggler pulls across prompt-sharded ranks: SpecActor's tail migration
on the real engines.

The reference lets a fully drained worker group adopt stragglers before it
offers itself to Best-of-N (``sim.py:952-958`` ``drained``): from the group
with the most live requests -- at least ``moved + 2`` of them, ties to the
first group -- it takes the live request with the lowest (acceptance-rate
estimate, id), and repeats while a source qualifies (``sim.py:546-593``
``pull_straggler``).  Here a group is a rank (one GPU, one
:class:`~paper_2511_16193_b200.engine.RolloutEngine` over its prompt shard)
and the move is real data: token row, lengths, budget, KV pages and the
drafter's per-slot state over NCCL P2P (``migrate.send_requests`` /
``recv_requests``; host-staged over gloo for one-GPU runs).

:class:`StragglerPull` is a :class:`~paper_2511_16193_b200.policy.RolloutDriver`
hook: every ``interval`` steps (and continuously once the rank is drained)
the driver stops with no step in flight and the ranks exchange their live
sets (one ``all_gather_object``), compute the same moves from
:func:`plan_pulls`, and run them pair by pair in plan order.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ConfigError


@dataclass(frozen=True)
class Move:
    src: int
    src_slot: int
    dst: int
    dst_slot: int
    request_id: int


def plan_pulls(states: list[dict]) -> list[Move]:
    """Moves for one exchange.  ``states[r]`` = ``{"live": [(slot, request
    id, estimate), ...], "free": [slot, ...]}`` of rank r, optionally with
    ``"n_live"`` when ``live`` lists only the slowest candidates.  Ranks with
    no live request are targets, in rank order; each adopts stragglers by
    the reference rule until no source has ``moved + 2`` live requests or it
    has no free slot left."""
    live = {r: list(st["live"]) for r, st in enumerate(states)}
    n_live = {r: int(st.get("n_live", len(st["live"]))) for r, st in enumerate(states)}
    free = {r: list(st["free"]) for r, st in enumerate(states)}
    targets = [r for r in range(len(states)) if n_live[r] == 0]
    moves: list[Move] = []
    for t in targets:
        moved = 0
        while free[t]:
            best = None
            for r in range(len(states)):
                if r == t or r in targets or not live[r]:
                    continue
                if n_live[r] >= moved + 2 and (best is None or n_live[r] > n_live[best]):
                    best = r
            if best is None:
                break
            slot, rid, _ = min(live[best], key=lambda x: (x[2], x[1]))
            live[best] = [x for x in live[best] if x[0] != slot]
            n_live[best] -= 1
            moves.append(Move(best, slot, t, free[t].pop(0), rid))
            moved += 1
    return moves


# one rank's exchange record: n_live, n_free, CAND x (slot, id, estimate), CAND free slots
CAND = 16
REC = 2 + 3 * CAND + CAND


def encode_state(live: list, free: list):
    import torch

    t = torch.full((REC,), -1.0, dtype=torch.float64)
    t[0], t[1] = len(live), len(free)
    for i, (slot, rid, est) in enumerate(sorted(live, key=lambda x: (x[2], x[1]))[:CAND]):
        t[2 + 3 * i: 5 + 3 * i] = torch.tensor([slot, rid, est], dtype=torch.float64)
    for i, slot in enumerate(free[:CAND]):
        t[2 + 3 * CAND + i] = slot
    return t


def decode_state(t) -> dict:
    v = t.tolist()
    n_live, n_free = int(v[0]), int(v[1])
    live = [(int(v[2 + 3 * i]), int(v[3 + 3 * i]), v[4 + 3 * i]) for i in range(min(n_live, CAND))]
    free = [int(v[2 + 3 * CAND + i]) for i in range(min(n_free, CAND))]
    return {"live": live, "n_live": n_live, "free": free}


class StragglerPull:
    """Driver hook running :func:`plan_pulls` across ranks.

    ``requests_by_id`` maps every request id of the job to its reference
    ``Request`` (all ranks build the same trace), so an adopting rank knows
    the request's reference fields.  ``interval``: steps between exchanges
    while the rank still has live requests."""

    def __init__(self, dist, requests_by_id: dict, interval: int = 16):
        if interval < 1:
            raise ConfigError("straggler exchange interval must be >= 1")
        self.dist, self.by_id, self.interval = dist, requests_by_id, interval
        self.moves: list[Move] = []
        self.bytes_moved = 0
        self.exchanges = 0

    def warmup(self, device) -> None:
        """Create the P2P communicators every rank pair may use before the
        timed rollout: NCCL builds a pair's communicator lazily on its first
        send/recv, which costs far more than a move."""
        dist = self.dist
        rank, world = dist.get_rank(), dist.get_world_size()
        dev = "cpu" if dist.get_backend() == "gloo" else device
        t = torch.zeros(4, dtype=torch.int32, device=dev)
        for a in range(world):
            for b in range(a + 1, world):
                if rank == a:
                    dist.send(t, b)
                    dist.batch_isend_irecv([dist.P2POp(dist.isend, t, b)])[0].wait()
                elif rank == b:
                    dist.recv(t, a)
                    dist.batch_isend_irecv([dist.P2POp(dist.irecv, t, a)])[0].wait()
        recs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(recs, t)

    def __call__(self, driver, local_done: bool, t_ms: float, events: list, can_run: bool = True) -> bool:
        """One exchange at a quiescent point; returns False once every rank
        is done (the driver then stops).  A rank out of steps (``can_run``
        False) offers no free slots: it could not run adopted requests."""
        dist = self.dist
        rank = dist.get_rank()
        live, free = driver.slot_states()
        if not can_run:
            free = []
        # one fixed-size record per rank, one all_gather (device tensors
        # over NCCL, host over gloo): ~tens of us, unlike all_gather_object
        mine = encode_state([] if local_done else live, free)
        if dist.get_backend() != "gloo":
            mine = mine.to(driver.eng.dev)
        recs = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
        dist.all_gather(recs, mine)
        states = [decode_state(r.cpu()) for r in recs]
        self.exchanges += 1
        moves = plan_pulls(states)
        pairs: dict[tuple[int, int], list[Move]] = {}
        for mv in moves:
            pairs.setdefault((mv.src, mv.dst), []).append(mv)
        from .migrate import recv_requests, send_requests

        for (src, dst), mvs in pairs.items():
            if rank == src:
                for mv in mvs:
                    driver.release_slot(mv.src_slot)
                self.bytes_moved += send_requests(dist, driver.eng, [mv.src_slot for mv in mvs], dst)
                for mv in mvs:
                    driver.log_event(events, t_ms, "migrate", f"rank-{src}", mv.request_id, {"to": f"rank-{dst}"})
            elif rank == dst:
                for mv in mvs:
                    driver.stash_slot(mv.dst_slot)
                recv_requests(dist, driver.eng, [mv.dst_slot for mv in mvs], src)
                for mv in mvs:
                    driver.adopt_slot(mv.dst_slot, self.by_id[mv.request_id])
        self.moves += moves
        # keep going while any rank has work (after this exchange's moves)
        busy = sum(st["n_live"] for st in states) > 0
        return busy
