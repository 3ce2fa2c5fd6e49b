"""Benchmark of the B200 speculative-rollout hot path (BASELINE.json metric:
rollout accepted tokens/s; mean accepted length; roofline %).

Workload (BASELINE.json configs[1]): Qwen2.5-1.5B-shaped random-init target,
256 prompts per GPU, k=4 n-gram drafter (vLLM prompt-lookup semantics,
min_n=1, max_n=3), greedy exact-match verification, bonus token on.  Prompt
lengths come from the reference trace generator (default_trace_spec: U[128,
1024]), prompt tokens from the keyed stream (seed, rid, "prompt").  A step is
one speculation window over the whole batch: n-gram draft -> verify forward
(M = 256 x 5 rows through 28 layers + lm_head with fused argmax) -> accept /
commit.  The batch is kept full (no request reaches its budget during the
run), i.e. steady-state throughput.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 runs under torchrun, one rank per GPU, 256 prompts per rank (weak
scaling by prompt sharding, no data-path collective).  Timing: CUDA events
on the launching stream, barrier + synchronize on both sides, max over ranks.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import re
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MODEL = "qwen2.5-1.5b"
BATCH = 256
K = 4
METRIC = "rollout accepted tokens/sec (Qwen2.5-1.5B-shaped target, batch 256/GPU, k=4, greedy)"
UNIT = "tokens/s"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=BATCH, help="prompts per GPU")
    ap.add_argument("--model", default=MODEL)
    ap.add_argument("--layers", type=int, default=None, help="debug only: truncate depth")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="launch every kernel from the host instead of replaying a CUDA graph")
    ap.add_argument("--drafter", choices=["synthetic", "ngram"], default="synthetic",
                    help="synthetic: reference accept_draw law over the target's own greedy "
                         "continuation (SURVEY 7.1e); ngram: vLLM prompt lookup")
    ap.add_argument("--accept-method", default="draft-0.5b",
                    help="reference drafting method whose latent acceptance/keyed draws drive the "
                         "synthetic drafter (scenarios.METHODS)")
    return ap.parse_args()


# -- workload -------------------------------------------------------------------


def workload(rank: int, batch: int, steps_total: int, vocab: int, world: int = 1):
    from paper_2511_16193_b200 import scenarios
    from paper_2511_16193_b200.dist import shard
    from paper_2511_16193_b200.streams import stream
    from paper_2511_16193_b200.workload import gen_trace

    # global batch of batch*world prompts, round-robin over ranks (sim.py:307-309)
    trace = shard(gen_trace(scenarios.default_trace_spec(batch=batch * world, seed=0)), rank, world)
    prompts = [stream(0, r.id, "prompt").integers(0, vocab, size=r.prompt_len).astype(np.int32)
               for r in trace]
    # budget large enough that no request leaves the batch during the run
    budget = 8 + (K + 1) * steps_total
    return trace, prompts, [budget] * len(trace)


# -- clocks -----------------------------------------------------------------------


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# -- our arm -------------------------------------------------------------------------


def traffic_bytes():
    f = ROOT / "profiles" / "r01" / "ncu_step_layer0.json"
    try:
        for d in json.loads(f.read_text()):
            m = re.search(r"gemm_\w*kernel<(\d+), (\d+)", d["kernel"])
            if m and m.group(2) == "2":  # epilogue 2 = SwiGLU: the gate_up GEMM
                return d["dram_read_bytes"] + d["dram_write_bytes"]
    except Exception:
        return None
    return None


def peaks():
    if PEAKS.exists():
        d = json.loads(PEAKS.read_text())
        return d["bf16_tflops"], d["bf16_tflops_sustained"], d["hbm_gbs"], "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def workload_config(args, s, world):
    """The bench's workload description, shared by both arms."""
    B = args.batch
    return {"workload": f"configs[1]: {args.model}-shaped target, batch {B}/GPU, k={K}, "
                        f"single {args.drafter} drafter, greedy exact match, bonus token",
            "model": args.model, "layers": s.layers, "batch_per_gpu": B, "global_batch": B * world,
            "k": K, "verify_rows_per_step": B * (K + 1), "prompt_len": "U[128,1024] (default_trace_spec)",
            "parallelism": f"prompt-sharded x{world} (no data-path collective)",
            "l2": "inputs larger than L2 (3.1 GB weights + paged KV per step)",
            "cuda_graph": not args.eager}


def run_ours(args, rank, world, dist):
    import torch

    from paper_2511_16193_b200 import _native
    from paper_2511_16193_b200.engine import NgramDrafter, RolloutEngine, SyntheticDrafter
    from paper_2511_16193_b200.model import DeviceModel, init_weights, shape

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    lib = _native.lib()
    s = shape(args.model, args.layers)
    steps_total = args.warmup + 3 * args.steps + 12
    trace, prompts, budget = workload(rank, args.batch, steps_total, s.vocab, world)
    max_len = max(len(p) for p in prompts) + budget[0] + K + 8
    big = s.linear_params() > 20e9   # fp32 + bf16 copies would not fit: convert layer by layer
    w = init_weights(s, seed=0, device="cuda", lazy=big)
    B = len(prompts)
    model = DeviceModel(s, w, dtype="bf16", max_requests=B, max_len=max_len,
                        max_tokens=B * (K + 1), max_seqs=B)
    del w
    torch.cuda.empty_cache()
    # untimed: the target's greedy continuation (plain decode), which the
    # synthetic drafter proposes under the reference's keyed acceptance law
    plain = RolloutEngine(model, prompts, budget, k=0, history=1)
    plain.prefill()
    plain.run()
    truth = plain.outputs()
    ngram_probe = None
    if args.drafter == "synthetic":
        drafter = SyntheticDrafter(truth, trace, args.accept_method, seed=0)
        ngram_probe = probe_ngram(RolloutEngine, NgramDrafter, model, prompts, budget, truth)
    else:
        drafter = NgramDrafter(1, 3)
    del plain
    eng = RolloutEngine(model, prompts, budget, k=K, drafters=(drafter,), bonus_token=True, history=1)
    eng.prefill()
    if not args.eager:
        eng.capture()
    clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", 0))).__enter__()
    for _ in range(args.warmup):
        eng.step()
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- timed region: K device-resident steps (inputs already in HBM)
    hist = torch.zeros((args.steps, B, 4), dtype=torch.int32, device="cuda")
    gen0 = eng.gen_len.sum()
    launches0 = lib.sr_launch_count()
    lib.sr_model_profile(model.handle, 1 if args.eager else 0, None, None)
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(st)
    for i in range(args.steps):
        eng.step()
        hist[i].copy_(eng.history[0])
    ev1.record(st)
    barrier()
    clocks.__exit__(None, None, None)
    launches = lib.sr_launch_count() - launches0
    ms = ev0.elapsed_time(ev1)
    committed = int((eng.gen_len.sum() - gen0).item())
    cat_ms = (ctypes.c_float * 8)()
    cat_n = (ctypes.c_int32 * 8)()
    lib.sr_model_profile(model.handle, 0, cat_ms, cat_n)
    if not args.eager:
        # kernel durations: a second graph of the same step with CUDA event
        # nodes bracketing every launch (captured on the launching stream);
        # replayed after the timed region, read back from its last replay
        lib.sr_model_profile(model.handle, 1, None, None)
        l0 = lib.sr_launch_count()
        prof_graph = eng.capture(install=False)
        per_step_launches = lib.sr_launch_count() - l0
        for _ in range(3):
            prof_graph.replay()
        torch.cuda.synchronize()
        _native.check(lib.sr_model_profile(model.handle, 0, cat_ms, cat_n), "sr_model_profile")
        launches = int(per_step_launches * args.steps)  # every replay launches them once
        for i in range(8):
            cat_ms[i] *= args.steps
        del prof_graph
    outs_ok = all(o == t[: len(o)] for o, t in zip(eng.outputs(), truth))
    h = hist.cpu().numpy().reshape(-1, 4)
    live = h[h[:, 0] + h[:, 2] > 0]
    accepted_mean = float(live[:, 1].mean()) if len(live) else 0.0
    committed_per_window = float(live[:, 2].mean()) if len(live) else 0.0
    proposed_mean = float(live[:, 0].mean()) if len(live) else 0.0

    # ---- e2e: same steps through the public API with host buffers each step
    budget_h = torch.tensor(budget, dtype=torch.int32).pin_memory()
    out_h = torch.empty((B, 4 + K + 2), dtype=torch.int32).pin_memory()
    e2e_in = budget_h.numel() * 4
    e2e_out = out_h.numel() * 4
    lib.sr_model_profile(model.handle, 0, None, None)
    gen1 = eng.gen_len.sum()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.eager:
        e0.record(st)
        for _ in range(args.steps):
            eng.max_new.copy_(budget_h, non_blocking=True)      # H2D: per-step request budgets
            seq_before = eng.seq_len.clone()
            eng.step()
            idx = (seq_before[:, None] + torch.arange(K + 2, device="cuda")[None, :]).clamp(max=eng.stride - 1)
            res = torch.cat([eng.history[0], torch.gather(eng.tokens, 1, idx.long())], 1)
            out_h.copy_(res, non_blocking=True)                 # D2H: outcomes + new tokens
            st.synchronize()
        e1.record(st)
    else:
        # the public API's host-facing step: H2D budgets -> step -> D2H results,
        # one graph per step over two result buffers; the host reads step i's
        # result (waiting on its event) while step i+1 runs -- every step's
        # result is read inside the timed region
        out2 = [out_h, torch.empty_like(out_h).pin_memory()]
        graphs = [eng.capture_io(budget_h, o) for o in out2]
        done = [torch.cuda.Event(), torch.cuda.Event()]
        check_sum = 0
        e0.record(st)
        for i in range(args.steps):
            eng.step_io(graphs[i % 2])
            done[i % 2].record(st)
            if i > 0:
                done[(i - 1) % 2].synchronize()
                check_sum += int(out2[(i - 1) % 2][0, 2])       # host reads step i-1's result
        done[(args.steps - 1) % 2].synchronize()
        check_sum += int(out2[(args.steps - 1) % 2][0, 2])
        e1.record(st)
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    e2e_committed = int((eng.gen_len.sum() - gen1).item())
    # drift check: the e2e steps run on contexts ~(K + 3) * tokens/window
    # longer than the device-timed ones; the same device replay after them
    # separates that from the host-facing overhead
    gen2 = eng.gen_len.sum()
    barrier()
    ev0.record(st)
    for _ in range(args.steps):
        eng.step()
    ev1.record(st)
    barrier()
    after_ms = ev0.elapsed_time(ev1)
    after_committed = int((eng.gen_len.sum() - gen2).item())

    # ---- cross-rank reduction: max time, summed tokens
    from paper_2511_16193_b200.dist import reduce_step_stats

    (ms_max, e2e_max, after_max), (tot_committed, tot_e2e, tot_after) = reduce_step_stats(
        [ms, e2e_ms, after_ms], [committed, e2e_committed, after_committed], dist, device="cuda")

    # ---- roofline of the dominant kernel family: the verify GEMMs (tensor-bound)
    gemm_ms = sum(cat_ms[i] for i in range(5))
    rows = B * (K + 1)
    flops_step = 2.0 * rows * s.linear_params()
    burst, sustained, hbm, src = peaks()
    achieved = flops_step * args.steps / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    attn_ms = cat_ms[5] + cat_ms[7]
    step_ms = ms / args.steps
    result = {
        "metric": METRIC, "value": tot_committed / (ms_max * 1e-3), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init N(0,0.02) weights; keyed-stream prompt tokens; reference trace lengths)",
        "config": workload_config(args, s, world),
        "mean_accepted_length": accepted_mean,
        "drafter": (f"synthetic: target's greedy continuation, accepted iff reference keyed "
                    f"accept_draw u < latent_accept['{args.accept_method}'] (sim.py:322-336)"
                    if args.drafter == "synthetic" else "n-gram (vLLM prompt lookup, min_n=1, max_n=3)"),
        "outputs_equal_plain_greedy": outs_ok,
        "ngram_probe": ngram_probe,
        "mean_proposed": proposed_mean,
        "tokens_per_window": committed_per_window,
        "roofline": {"bound": "tensor", "kernel": "verify GEMMs (qkv, o, gate_up+SwiGLU, down, lm_head+argmax)",
                     "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
                     "frac": (achieved / sustained) if achieved else None,
                     "peak_source": f"{src} bf16_tflops_sustained (kernels timed inside the step)",
                     "traffic": traffic_bytes(),
                     "traffic_note": "DRAM read+write bytes per launch of the largest verify GEMM (gate_up "
                                     "+SwiGLU) from profiles/r01/ncu_step_layer0.json (ncu --set full); "
                                     "algorithmic = 55.0 MB weights + 3.9 MB activations in + 22.9 MB "
                                     "SwiGLU output (written to L2, consumed there by down: DRAM sees "
                                     "weights + activations + a partial write-back)",
                     "algorithmic_flops_per_step": flops_step,
                     "gemm_ms_per_step": gemm_ms / args.steps,
                     "gemm_share_of_step": (gemm_ms / args.steps) / step_ms,
                     "attention_ms_per_step": attn_ms / args.steps,
                     "attention_combine_ms_per_step": cat_ms[7] / args.steps,
                     "other_ms_per_step": cat_ms[6] / args.steps,
                     "per_gemm_ms_per_step": {n: cat_ms[i] / args.steps for i, n in
                                              enumerate(["qkv", "o", "gate_up", "down", "lm_head"])}},
        "e2e": {"value": tot_e2e / (e2e_max * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": e2e_in, "d2h_bytes_per_step": e2e_out,
                "device_value_after": tot_after / (after_max * 1e-3),
                "note": "device_value_after = the device-resident replay of the same number of steps run "
                        "right after the e2e steps (longer contexts): e2e vs it is the host-facing cost"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
    }
    return result, (s, model, prompts)


def probe_ngram(RolloutEngine, NgramDrafter, model, prompts, budget, truth, steps=8):
    """Measured acceptance of the real n-gram drafter on this workload (not timed)."""
    import torch

    eng = RolloutEngine(model, prompts, budget, k=K, drafters=(NgramDrafter(1, 3),), bonus_token=True,
                        history=steps)
    eng.prefill()
    for _ in range(steps):
        eng.step()
    torch.cuda.synchronize()
    h = eng.outcome_rows().reshape(-1, 4)
    live = h[h[:, 0] + h[:, 2] > 0]
    same = all(o == t[: len(o)] for o, t in zip(eng.outputs(), truth))
    return {"steps": steps, "mean_proposed": float(live[:, 0].mean()), "mean_accepted": float(live[:, 1].mean()),
            "tokens_per_window": float(live[:, 2].mean()), "outputs_equal_plain_greedy": same}


# -- CPU baseline (oracle port of the same path) ----------------------------------------


def cpu_baseline(s, model, prompts, requests=8, prompt_cap=128, windows=24):
    """Bounded sample of the same workload through the CPU oracle port."""
    import torch

    from oracle.qwen2_oracle import CachedRollout, Qwen2Oracle

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    w = weights_to_cpu(s, model)
    runner = CachedRollout(Qwen2Oracle(s, w, "bf16"))
    ps = [p[:prompt_cap].tolist() for p in prompts[:requests]]
    seqs = runner.prefill(ps)
    t0 = time.perf_counter()
    committed = 0
    for _ in range(windows):
        for r in range(requests):
            c, _, _ = runner.step(r, seqs[r], K)
            committed += c
    dt = time.perf_counter() - t0
    return {"value": committed / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{requests} requests x {windows} windows (k={K}, n-gram) of the full "
                      f"{s.layers}-layer {s.name} model on CPU (oracle/qwen2_oracle.py CachedRollout, "
                      f"bf16-emulated torch, prompts truncated to {prompt_cap} tokens), {dt:.1f} s"}


def weights_to_cpu(s, model):
    """Canonical fp32 weights rebuilt from the device model (identical values)."""
    from paper_2511_16193_b200.model import pair_deinterleave_heads
    w = {"embed": model.embed.float().cpu(), "final_norm": model.final_norm.cpu(), "layers": []}
    w["lm_head"] = w["embed"] if s.tied else model.lm_head.float().cpu()
    nq, nkv, hd, I = s.q_heads * s.head_dim, s.kv_heads * s.head_dim, s.head_dim, s.intermediate
    def unpair(x, heads):
        return pair_deinterleave_heads(x, heads, hd) if model.fused_rope else x

    for t in model.layer_tensors:
        qkv, b = t["w_qkv"].float().cpu(), t["b_qkv"].cpu()
        gu = t["w_gu"].float().cpu().view(I // 16, 2, 16, s.hidden)
        w["layers"].append({
            "ln1": t["ln1"].cpu(), "ln2": t["ln2"].cpu(),
            "wq": unpair(qkv[:nq], s.q_heads), "wk": unpair(qkv[nq:nq + nkv], s.kv_heads), "wv": qkv[nq + nkv:],
            "bq": unpair(b[:nq], s.q_heads), "bk": unpair(b[nq:nq + nkv], s.kv_heads), "bv": b[nq + nkv:],
            "wo": t["w_o"].float().cpu(), "wg": gu[:, 0].reshape(I, s.hidden),
            "wu": gu[:, 1].reshape(I, s.hidden), "wd": t["w_down"].float().cpu()})
    return w


def run_reference(args):
    """The reference arm: the CPU implementation of the path (oracle port;
    the reference itself is a Python simulator with no model arithmetic)."""
    import torch

    from paper_2511_16193_b200.model import init_weights, shape

    s = shape(args.model, args.layers)
    torch.set_num_threads(os.cpu_count() or 1)
    _, prompts, _ = workload(0, args.batch, 1, s.vocab)
    from oracle.qwen2_oracle import CachedRollout, Qwen2Oracle

    w = init_weights(s, seed=0, device="cpu")
    runner = CachedRollout(Qwen2Oracle(s, w, "bf16"))
    del w
    reqs = 2
    seqs = runner.prefill([p[:128].tolist() for p in prompts[:reqs]])
    for _ in range(max(args.warmup, 1)):
        for r in range(reqs):
            runner.step(r, seqs[r], K)
    times, committed = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        for r in range(reqs):
            c, _, _ = runner.step(r, seqs[r], K)
            committed += c
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = committed / total
    sample = (f"{reqs} requests x {args.steps} windows (k={K}, n-gram) through the full {s.layers}-layer "
              f"{s.name} model, oracle port (torch CPU, bf16-emulated), prompts truncated to 128 tokens")
    return {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic", "config": workload_config(args, s, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count() or 1, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    result, ctx = run_ours(args, rank, world, dist)
    if rank == 0:
        from paper_2511_16193_b200.model import shape
        # the CPU sample of a >10B model would need its fp32 weights in host RAM
        if world == 1 and not args.no_cpu_baseline and shape(args.model).linear_params() <= 10e9:
            result["cpu_baseline"] = cpu_baseline(*ctx)
        else:
            result["cpu_baseline"] = None
        print(json.dumps(result), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
