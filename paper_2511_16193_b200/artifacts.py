"""Reference-compatible run artifacts, so the reference's CLI
and notebooks can analyse B200 runs:

* ``write_samples`` -- measured step latencies as the ``fit`` command's input
  (CSV with columns ``b,latency_ms,key``; keys ``draft/<method>/<g_d>``,
  ``verify/<config>/<w>``, ``plain/<config>``; reference ``cli.py:290-310``);
* ``write_simulation`` -- a ``simulate`` run as ``summary.json``,
  ``requests.csv``, ``workers.csv`` and ``events.jsonl`` (reference
  ``cli.py:473-487``: floats with 6 decimals, sorted-key JSON, one event
  object per line).
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

REQUEST_COLUMNS = ["request", "true_len", "finish_ms", "committed", "drafted", "wasted",
                   "windows", "partial_events", "winner", "tokens_per_window"]
WORKER_COLUMNS = ["worker", "role", "busy_ms", "idle_ms", "drained_ms"]


def _cell(x) -> str:
    return f"{x:.6f}" if isinstance(x, float) else str(x)


def _csv(path: Path, columns: list[str], rows) -> None:
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(columns)
        for row in rows:
            w.writerow([_cell(x) for x in row])


def write_samples(path, samples) -> None:
    """``samples``: iterable of ``costmodel.ProfileSample`` (b, latency_ms, key)."""
    _csv(Path(path), ["b", "latency_ms", "key"], ([s.b, float(s.latency_ms), s.key] for s in samples))


def write_simulation(metrics, out_dir) -> list[Path]:
    """Write a ``SimMetrics`` in the reference CLI's ``simulate`` layout."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    m = metrics
    summary = {"policy": m.policy, "seed": m.seed, "makespan_ms": round(m.makespan_ms, 6),
               "total_committed": m.total_committed, "total_wasted": m.total_wasted,
               "mean_tgs": round(m.mean_tgs, 6), "bon_assign_count": m.bon_assign_count,
               "reconfig_count": m.reconfig_count}
    paths = [out / "summary.json", out / "requests.csv", out / "workers.csv", out / "events.jsonl"]
    with open(paths[0], "w", encoding="utf-8") as fh:
        json.dump(summary, fh, indent=2, sort_keys=True)
        fh.write("\n")
    _csv(paths[1], REQUEST_COLUMNS,
         ([r.id, r.true_len, r.finish_ms, r.committed, r.drafted, r.wasted, r.windows, r.partial_events,
           r.winner, r.tokens_per_window] for r in m.requests.values()))
    _csv(paths[2], WORKER_COLUMNS,
         ([w.id, w.role, w.busy_ms, w.idle_ms, w.drained_ms]
          for w in sorted(m.workers.values(), key=lambda w: w.id)))
    with open(paths[3], "w", encoding="utf-8") as fh:
        for ev in m.events:
            fh.write(json.dumps(ev, sort_keys=True) + "\n")
    return paths
