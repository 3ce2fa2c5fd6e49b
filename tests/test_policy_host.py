"""Host logic of the engine-side policy loop (CPU): the batched outcome rings
follow the reference estimator (workload.py:42-56) exactly."""

from __future__ import annotations

import numpy as np


def test_outcome_rings_match_reference_estimator():
    from paper_2511_16193_b200.policy import OutcomeRings
    from paper_2511_16193_b200.workload import AcceptanceEstimator

    rng = np.random.default_rng(0)
    B, N, W = 5, 3, 8
    rings = OutcomeRings(B, N, W, [0.75, 0.5, 0.88])
    ref = [[AcceptanceEstimator(W, p) for p in (0.75, 0.5, 0.88)] for _ in range(B)]
    for _ in range(30):
        mask = rng.random((B, N)) < 0.6
        prop = rng.integers(0, 5, (B, N))
        acc = np.minimum(prop, rng.integers(0, 5, (B, N)))
        rings.record(mask, prop, acc)
        for b, n in zip(*np.nonzero(mask)):
            ref[b][n].record(int(prop[b, n]), int(acc[b, n]))
        est = rings.estimate()
        for b in range(B):
            for n in range(N):
                assert est[b, n] == ref[b][n].estimate()
                assert rings.estimator(b, n).estimate() == ref[b][n].estimate()
                assert rings.estimator(b, n).count() == ref[b][n].count()


def test_choose_placement_picks_higher_modeled_throughput():
    """Both reference plan searches run; the placement is the mode with the
    higher estimate (coupled on the B200 calibration)."""
    from pathlib import Path

    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.costmodel import CostModel
    from paper_2511_16193_b200.policy import choose_placement

    cm = CostModel.load(Path(__file__).resolve().parent.parent / "profiles" / "r01" / "costmodel_b200.json")
    pl = choose_placement(256, cm, 0.7, "ngram")
    assert pl.mode == "coupled"
    assert pl.tgs_estimate == pl.coupled.tgs_estimate >= pl.decoupled.tgs_estimate
    ref = scenarios.default_cost_model()
    pr = choose_placement(256, ref, 0.7)
    assert pr.tgs_estimate == max(pr.coupled.tgs_estimate, pr.decoupled.tgs_estimate)
