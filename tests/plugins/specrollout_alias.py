"""pytest plugin: serve this package under the reference's import name.

``python -m pytest -p specrollout_alias <reference pkg/tests>`` runs the
reference's OWN test files (never copied into this repo) against
``paper_2511_16193_b200``: ``import specrollout`` and every
``specrollout.<module>`` resolve to this build's modules of the same name.

Two test-only adjustments, both explicit:
* ``specrollout.cli`` is out of scope; a stub module carries its
  exit-code constants so test_acceptance.py imports, and the CLI-driven tests
  are deselected by the caller.
* Without a GPU, ``simulate()``'s per-window verification and
  ``generate_true_sequence`` are served by the CPU oracle
  (``oracle/rollout_oracle``, the test seam); with a GPU the device paths run
  as in the product.
"""

from __future__ import annotations

import sys
import types
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2511_16193_b200 as _pkg  # noqa: E402
from paper_2511_16193_b200 import (bon, costmodel, errors, planner, scenarios, sim, streams,  # noqa: E402
                                   workload)

sys.modules["specrollout"] = _pkg
for _name, _mod in dict(bon=bon, costmodel=costmodel, errors=errors, planner=planner, scenarios=scenarios,
                        sim=sim, streams=streams, workload=workload).items():
    sys.modules[f"specrollout.{_name}"] = _mod
    setattr(_pkg, _name, _mod)

_cli = types.ModuleType("specrollout.cli")
_cli.EXIT_OK, _cli.EXIT_CONFIG, _cli.EXIT_RUNTIME = 0, 2, 3


def _no_cli(*_a, **_k):
    raise NotImplementedError("the reference CLI is out of this build's scope (SURVEY §2)")


_cli.main = _no_cli
sys.modules["specrollout.cli"] = _cli


def _gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


if not _gpu():
    from oracle.rollout_oracle import OracleVerifier, true_tokens

    def _truth(request_id, true_len, seed):
        return [int(t) for t in true_tokens(seed, request_id, true_len)]

    sim.generate_true_sequence = _truth
    _pkg.generate_true_sequence = _truth

    _device_simulate = sim.simulate

    def _simulate(config, verifier_factory=None):
        return _device_simulate(config, verifier_factory=verifier_factory or OracleVerifier)

    sim.simulate = _simulate
    _pkg.simulate = _simulate
