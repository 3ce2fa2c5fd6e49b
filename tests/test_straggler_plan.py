"""Straggler-pull decisions (``straggler.plan_pulls``) against the
reference rule ``sim.py:546-593``: a drained rank adopts, from the rank with
the most live requests (>= moved + 2, ties to the lowest rank), the live
request with the lowest (estimate, id), repeatedly."""

from __future__ import annotations

from paper_2511_16193_b200.straggler import Move, plan_pulls


def st(live, free=()):
    return {"live": list(live), "free": list(free)}


def test_drained_rank_pulls_slowest_from_busiest():
    states = [st([], free=[0, 1, 2]),
              st([(0, 10, 0.9), (1, 11, 0.2), (2, 12, 0.5)]),
              st([(0, 20, 0.1), (1, 21, 0.3)])]
    # busiest is rank 1 (3 live): takes its slowest (id 11); then rank 1 has 2
    # live and rank 2 has 2 live: neither has moved + 2 = 3 -> stop
    assert plan_pulls(states) == [Move(1, 1, 0, 0, 11)]


def test_repeated_pulls_need_moved_plus_two():
    live = [(b, 100 + b, 0.5 + 0.01 * b) for b in range(6)]
    states = [st([], free=[3, 4, 5, 6]), st(live)]
    moves = plan_pulls(states)
    # 6 live: moved 0 needs >= 2 -> pull; 5 >= 3 -> pull; 4 >= 4 -> pull; 3 < 5 -> stop
    assert [m.request_id for m in moves] == [100, 101, 102]
    assert [m.dst_slot for m in moves] == [3, 4, 5]


def test_ties_lowest_rank_and_lowest_id():
    states = [st([(0, 7, 0.5), (1, 3, 0.5)]), st([], free=[9]), st([(0, 1, 0.5), (1, 2, 0.5)])]
    # ranks 0 and 2 both have 2 live: the first (rank 0) wins; equal estimates -> lowest id (3)
    assert plan_pulls(states) == [Move(0, 1, 1, 9, 3)]


def test_no_free_slot_or_no_source():
    assert plan_pulls([st([], free=[]), st([(0, 1, 0.1), (1, 2, 0.2)])]) == []
    assert plan_pulls([st([], free=[0]), st([(0, 1, 0.1)])]) == []       # a single straggler stays put
    assert plan_pulls([st([(0, 1, 0.1)]), st([(0, 2, 0.1)])]) == []      # nobody drained


def test_two_targets_in_rank_order():
    live = [(b, b, 0.1 * b) for b in range(5)]
    states = [st([], free=[0]), st(live), st([], free=[0, 1])]
    moves = plan_pulls(states)
    # rank 0 (one free slot) takes id 0; rank 2 then takes id 1 (4 live >= 2), id 2 (3 >= 3), stops (2 < 4)
    assert [(m.dst, m.request_id) for m in moves] == [(0, 0), (2, 1), (2, 2)]


def test_exchange_record_round_trip_keeps_slowest_candidates():
    from paper_2511_16193_b200.straggler import CAND, decode_state, encode_state

    live = [(b, 1000 + b, 1.0 - 0.01 * b) for b in range(40)]
    st = decode_state(encode_state(live, [3, 7]))
    assert st["n_live"] == 40 and st["free"] == [3, 7]
    assert [x[1] for x in st["live"]] == [1039 - i for i in range(CAND)]   # the CAND slowest
    full = [{"live": [], "free": [0, 1, 2]}, {"live": live, "free": [3, 7]}]
    short = [decode_state(encode_state([], [0, 1, 2])), st]
    assert plan_pulls(full) == plan_pulls(short)
