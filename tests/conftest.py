"""Test configuration: the ``gpu`` marker and shared helpers.

``-m "not gpu"`` runs on CPU: oracle vs golden fixtures, host logic, ABI
load.  ``-m gpu`` runs the CUDA path against the oracle (needs a B200).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


def golden(name: str):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def model():
    from paper_2511_16193_b200 import scenarios
    return scenarios.default_cost_model()


def make_trace(batch: int, seed: int, sigma: float | None = None):
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.workload import TraceSpec, gen_trace

    spec = scenarios.default_trace_spec(batch=batch, seed=seed)
    if sigma is not None:
        spec = TraceSpec(**{**spec.__dict__, "length_sigma": sigma})
    return gen_trace(spec)


def run_sim(model, trace, seed, verifier_factory=None, **kwargs):
    """The reference harness (pkg/tests/conftest.py:32-42) on our engine."""
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.sim import SimConfig, simulate

    opts = dict(trace=trace, model=model, method=scenarios.DEFAULT_METHOD, seed=seed,
                scale_cost=scenarios.default_scale_cost(),
                estimator_priors=scenarios.estimator_priors())
    opts.update(kwargs)
    return simulate(SimConfig(**opts), verifier_factory=verifier_factory)
