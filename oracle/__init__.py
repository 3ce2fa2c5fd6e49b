"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Restatements of the reference algorithms used as checkers by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg.  The
product package (``paper_2511_16193_b200``) never imports this directory.

Pinning:
  rollout_oracle  -- verify/commit semantics of pkg/src/specrollout/sim.py;
                     PINNED against golden runs of the reference itself
                     (tests/golden/sim_runs.json, keyed_draws.json).
  ngram_oracle    -- vLLM 0.22 NgramProposer semantics; PINNED against
                     golden outputs of vLLM's own function
                     (tests/golden/ngram_vllm.json).
  qwen2_oracle    -- PyTorch-CPU Qwen2 decoder arithmetic; the reference has
                     no model, so logits parity is UNPINNED by the reference
                     (cross-checked against transformers' Qwen2 instead).
"""
