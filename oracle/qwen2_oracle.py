"""CPU ORACLE (test infrastructure only) for the verification forward.

PyTorch-CPU restatement of the Qwen2-style decoder the GPU path runs
(paper_2511_16193_b200/csrc/model.cu).  The reference has no model at all --
its "target token" is a keyed random integer (sim.py:313-320) -- so logits
parity is UNPINNED by the reference; this oracle is cross-checked against
transformers' Qwen2ForCausalLM in tests/test_oracle_model.py instead.

Arithmetic (both modes): residual stream fp32; RMSNorm y = x*rsqrt(mean(x^2)+eps)*w
(bf16 mode: the GPU fuses the norm into the GEMMs, norm(x) W = r * (bf16(x*w) W),
so the rounding point is bf16(x*w) and r scales the fp32 accumulator);
RoPE on the NeoX halves with the shared float64->float32 cos/sin tables;
softmax in fp32.  In "bf16" mode values are rounded to bf16 exactly where the
GPU stores bf16: normed activations, rotated q/k and v (RoPE runs in the
qkv GEMM epilogue on the fp32 accumulator + bias), softmax probabilities
entering P.V, attention output, SwiGLU output.  GEMMs
accumulate in fp32 (double in "fp32" mode for a tighter reference).

Acceptance semantics for spec decoding follow sim.py:983-1042 (exact match,
optional bonus token) and vLLM's n-gram proposer (oracle/ngram_oracle.py).
"""

from __future__ import annotations

import numpy as np
import torch

from oracle import ngram_oracle, sampling_oracle


class Qwen2Oracle:
    def __init__(self, shape, weights: dict, dtype: str = "fp32"):
        from paper_2511_16193_b200.model import rope_tables

        self.s = shape
        self.bf16 = dtype == "bf16"
        cast = (lambda t: t.bfloat16().float()) if self.bf16 else (lambda t: t.double())
        self.acc = torch.float32 if self.bf16 else torch.float64
        w = weights
        self.embed = cast(w["embed"])
        self.lm_head = cast(w["lm_head"])
        self.final_norm = w["final_norm"].to(self.acc)
        self.layers = []
        for L in w["layers"]:
            self.layers.append({
                "ln1": L["ln1"].to(self.acc), "ln2": L["ln2"].to(self.acc),
                "wqkv": cast(torch.cat([L["wq"], L["wk"], L["wv"]], 0)),
                "bqkv": torch.cat([L["bq"], L["bk"], L["bv"]], 0).to(self.acc),
                "wo": cast(L["wo"]), "wg": cast(L["wg"]), "wu": cast(L["wu"]), "wd": cast(L["wd"]),
            })
        cos, sin = rope_tables(shape, 1 << 14)
        self.cos = torch.from_numpy(cos).to(self.acc)
        self.sin = torch.from_numpy(sin).to(self.acc)

    def accumulating_in(self, dtype) -> "Qwen2Oracle":
        """The same oracle (same weights, same bf16 rounding points) with its
        GEMMs / reductions accumulated in ``dtype``.  bf16 results depend on
        accumulation order, so comparing the fp32- and fp64-accumulating
        variants measures the spread any two bf16 implementations can show
        (the noise floor of GPU-vs-oracle bf16 parity)."""
        import copy

        o = copy.copy(self)
        for name in ("embed", "lm_head", "final_norm", "cos", "sin"):
            setattr(o, name, getattr(self, name).to(dtype))
        o.layers = [{k: v.to(dtype) for k, v in L.items()} for L in self.layers]
        o.acc = dtype
        return o

    def _r(self, t):
        return t.bfloat16().to(self.acc) if self.bf16 else t

    def _norm(self, x, w):
        var = (x * x).mean(-1, keepdim=True)
        return self._r(x * torch.rsqrt(var + self.s.rms_eps) * w)

    def _normed_proj(self, x, w, W):
        """norm(x, w) @ W.T with the GPU's rounding points (gemm.cuh NormArgs)."""
        if not self.bf16:
            return self._norm(x, w) @ W.t()
        r = torch.rsqrt((x * x).mean(-1, keepdim=True) + self.s.rms_eps)
        return r * (self._r(x * w) @ W.t())

    def _rope(self, x, pos):
        half = self.s.head_dim // 2
        c, s = self.cos[pos][:, None, :], self.sin[pos][:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return self._r(torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1))

    @torch.no_grad()
    def logits(self, tokens) -> torch.Tensor:
        """Causal forward over one full sequence; logits [L, V] (fp32/fp64)."""
        s = self.s
        T = len(tokens)
        pos = torch.arange(T)
        x = self.embed[torch.as_tensor(tokens, dtype=torch.long)].to(self.acc)
        nq, nkv, hd = s.q_heads, s.kv_heads, s.head_dim
        G = nq // nkv
        mask = torch.triu(torch.ones(T, T, dtype=torch.bool), 1)
        for L in self.layers:
            qkv = self._normed_proj(x, L["ln1"], L["wqkv"]) + L["bqkv"]
            q = qkv[:, : nq * hd].view(T, nq, hd)
            k = qkv[:, nq * hd: (nq + nkv) * hd].view(T, nkv, hd)
            v = self._r(qkv[:, (nq + nkv) * hd:].view(T, nkv, hd))
            q, k = self._rope(q, pos), self._rope(k, pos)
            k = k.repeat_interleave(G, dim=1)
            v = v.repeat_interleave(G, dim=1)
            sc = torch.einsum("qhd,khd->hqk", q, k) / float(np.sqrt(hd))
            sc = sc.masked_fill(mask, float("-inf"))
            m = sc.amax(-1, keepdim=True)
            p = torch.exp(sc - m)
            l = p.sum(-1, keepdim=True)
            o = torch.einsum("hqk,khd->qhd", self._r(p), v) / l.permute(1, 0, 2)
            x = x + self._r(o.reshape(T, nq * hd)) @ L["wo"].t()
            g = self._normed_proj(x, L["ln2"], L["wg"])
            u = self._normed_proj(x, L["ln2"], L["wu"])
            act = self._r(g / (1.0 + torch.exp(-g)) * u)
            x = x + act @ L["wd"].t()
        return self._normed_proj(x, self.final_norm, self.lm_head)

    def greedy(self, prompt, max_new: int) -> list[int]:
        """Plain greedy decode (lowest index on ties)."""
        seq = list(prompt)
        out = []
        for _ in range(max_new):
            tok = int(torch.argmax(self.logits(seq)[-1]))
            out.append(tok)
            seq.append(tok)
        return out

    def _pick(self, logits_row, pos: int, sample):
        """Greedy argmax, or the keyed sample (seed, request, temperature)."""
        if sample is None:
            return int(torch.argmax(logits_row))
        seed, req, temp = sample
        return sampling_oracle.sample(logits_row.float().numpy(), seed, req, pos, temp)

    def spec_decode(self, prompt, max_new: int, k: int, min_n: int = 1, max_n: int = 3,
                    bonus: bool = False, max_model_len: int | None = None, sample=None):
        """n-gram speculative decode with exact-match verification.

        ``sample`` = (seed, request row, temperature) switches the target token
        to the keyed Gumbel-max sample at each generated position.
        Returns (output tokens, outcome rows [(proposed, accepted, committed, wasted)]).
        """
        seq = list(prompt)
        out, rows = [], []
        # every generated token comes out of a window (the first window
        # starts from the last prompt token), as in sim.py:834-928
        while len(out) < max_new:
            remaining = max_new - len(out)
            d = ngram_oracle.propose(seq, min_n, max_n, k, max_model_len)[: min(k, remaining)]
            lg = self.logits(seq + d)
            y = [self._pick(lg[len(seq) - 1 + j], len(seq) + j, sample) for j in range(len(d) + 1)]
            a = 0
            while a < len(d) and d[a] == y[a]:
                a += 1
            n = len(d)
            if n == 0:
                c = 1
            elif a == n:
                c = n + (1 if bonus else 0)
            else:
                c = a + 1
            c = min(c, remaining)
            rows.append((n, a, c, 0 if a == n else max(n - a - 1, 0)))
            out += y[:c]
            seq += y[:c]
        return out, rows


    def spec_decode_bon(self, prompt, max_new: int, k: int, drafters, bonus: bool = False, sample=None):
        """Best-of-N speculative decode with exact-match verification.

        Every window, each of the N ``drafters`` (callables ``(seq, limit) ->
        draft tokens``) proposes from the same committed context; the target
        verifies each proposal (its token at every window position); the
        drafter with the longest accepted prefix wins, ties to the lowest
        index (incumbent first) -- the reference's first-finisher over
        replicas that share one committed sequence (sim.py:340-361; replicas
        from bon.py:79-139), collapsed into one window.  The winner's
        window commits by the reference rule (sim.py:983-1042).

        Returns (output tokens, windows, winners): ``windows[i]`` holds the N
        outcome rows (proposed, accepted, committed, wasted) of window i --
        losers commit 0 and waste their whole proposal, the winner wastes
        n - a - 1 on a partial accept (sim.py:1001-1010) -- and
        ``winners[i]`` the winning drafter index.
        """
        seq = list(prompt)
        out, windows, winners = [], [], []
        while len(out) < max_new:
            remaining = max_new - len(out)
            lim = min(k, remaining)
            res = []
            for dr in drafters:
                d = list(dr(list(seq), lim))[:lim]
                lg = self.logits(seq + d)
                y = [self._pick(lg[len(seq) - 1 + j], len(seq) + j, sample) for j in range(len(d) + 1)]
                a = 0
                while a < len(d) and d[a] == y[a]:
                    a += 1
                res.append((len(d), a, y))
            win = max(range(len(res)), key=lambda i: (res[i][1], -i))
            n, a, y = res[win]
            c = 1 if n == 0 else (n + (1 if bonus else 0) if a == n else a + 1)
            c = min(c, remaining)
            rows = []
            for i, (ni, ai, _) in enumerate(res):
                if i == win:
                    rows.append((ni, ai, c, 0 if ai == ni else max(ni - ai - 1, 0)))
                else:
                    rows.append((ni, ai, 0, ni))
            windows.append(rows)
            winners.append(win)
            out += y[:c]
            seq += y[:c]
        return out, windows, winners


def ngram_drafter(k: int, min_n: int = 1, max_n: int = 3, max_model_len: int | None = None):
    """Oracle n-gram drafter for :meth:`Qwen2Oracle.spec_decode_bon`."""
    return lambda seq, lim: ngram_oracle.propose(seq, min_n, max_n, k, max_model_len)[:lim]


class ModelDrafterOracle:
    """Oracle small-model drafter: ``limit`` autoregressive steps of a draft
    decoder from the committed context (greedy, or the keyed sample with the
    target's noise at the same output positions -- the GPU ModelDrafter's
    Gumbel coupling)."""

    def __init__(self, oracle: Qwen2Oracle, sample=None):
        self.o = oracle
        self.sample = sample

    def __call__(self, seq, lim):
        d = []
        for j in range(lim):
            lg = self.o.logits(seq + d)[-1]
            d.append(self.o._pick(lg, len(seq) + j, self.sample))
        return d


def margin(logits_row: torch.Tensor) -> float:
    """Gap between the top-1 and top-2 logit (tie safety of greedy parity)."""
    top = torch.topk(logits_row.double(), 2).values
    return float(top[0] - top[1])


class CachedRollout:
    """KV-cached CPU speculative rollout with the oracle's arithmetic: the CPU
    port of the hot path timed by bench.py's cpu_baseline / --impl reference
    legs (prefill once, then n-gram draft -> verify window -> exact-match
    accept per request, sim.py:983-1042 semantics)."""

    def __init__(self, oracle: Qwen2Oracle):
        self.o = oracle
        self.k_cache: list[list[torch.Tensor]] = []
        self.v_cache: list[list[torch.Tensor]] = []

    @torch.no_grad()
    def _forward(self, req: int, tokens, start: int) -> torch.Tensor:
        """Positions [start, start+len(tokens)) with cached keys [0, start)."""
        o, s = self.o, self.o.s
        T = len(tokens)
        pos = torch.arange(start, start + T)
        x = o.embed[torch.as_tensor(tokens, dtype=torch.long)].to(o.acc)
        nq, nkv, hd = s.q_heads, s.kv_heads, s.head_dim
        G = nq // nkv
        mask = torch.ones(T, start + T, dtype=torch.bool).triu(start + 1)
        for li, L in enumerate(o.layers):
            qkv = o._normed_proj(x, L["ln1"], L["wqkv"]) + L["bqkv"]
            q = o._rope(qkv[:, : nq * hd].view(T, nq, hd), pos)
            k = o._rope(qkv[:, nq * hd: (nq + nkv) * hd].view(T, nkv, hd), pos)
            v = o._r(qkv[:, (nq + nkv) * hd:].view(T, nkv, hd))
            kc = torch.cat([self.k_cache[req][li][:start], k]) if start else k
            vc = torch.cat([self.v_cache[req][li][:start], v]) if start else v
            self.k_cache[req][li], self.v_cache[req][li] = kc, vc
            kk, vv = kc.repeat_interleave(G, 1), vc.repeat_interleave(G, 1)
            sc = torch.einsum("qhd,khd->hqk", q, kk) / float(np.sqrt(hd))
            sc = sc.masked_fill(mask, float("-inf"))
            p = torch.exp(sc - sc.amax(-1, keepdim=True))
            l = p.sum(-1, keepdim=True)
            att = torch.einsum("hqk,khd->qhd", o._r(p), vv) / l.permute(1, 0, 2)
            x = x + o._r(att.reshape(T, nq * hd)) @ L["wo"].t()
            g = o._normed_proj(x, L["ln2"], L["wg"])
            u = o._normed_proj(x, L["ln2"], L["wu"])
            x = x + o._r(g / (1.0 + torch.exp(-g)) * u) @ L["wd"].t()
        return o._normed_proj(x, o.final_norm, o.lm_head)

    def prefill(self, prompts) -> list[list[int]]:
        seqs = []
        for p in prompts:
            self.k_cache.append([None] * len(self.o.layers))
            self.v_cache.append([None] * len(self.o.layers))
            lg = self._forward(len(seqs), list(p), 0)
            seqs.append(list(p) + [int(torch.argmax(lg[-1]))])
        return seqs

    def step(self, req: int, seq: list[int], k: int, min_n=1, max_n=3, bonus=True):
        """One speculation window for one request; returns committed tokens."""
        d = ngram_oracle.propose(seq, min_n, max_n, k)
        lg = self._forward(req, [seq[-1]] + d, len(seq) - 1)
        y = [int(t) for t in torch.argmax(lg, -1)]
        a = 0
        while a < len(d) and d[a] == y[a]:
            a += 1
        c = (len(d) + (1 if bonus else 0)) if a == len(d) and d else (a + 1)
        seq += y[:c]
        return c, len(d), a


class BatchedRollout:
    """Batched, KV-cached CPU port of the benched rollout step (bench.py's
    ``--impl reference`` arm and ``cpu_baseline``): every window of the batch
    goes through ONE forward -- the projections and MLP as GEMMs over all
    window rows, attention per request over its cache -- with the oracle's
    arithmetic, then exact-match acceptance with the reference's commit rule
    (sim.py:983-1042, bonus token on as in the bench).

    Drafts follow the bench's reference-acceptance law: the
    draft at output position g is the target's own greedy token ``truth[g]``
    (from this port's plain decode) when the reference's keyed acceptance
    uniform ``u[g] < p`` (sim.py:322-336), else a wrong token.

    Like the GPU path, the port must compute a position's token identically
    in a plain-decode step and in a speculation window, or its own greedy
    continuation would not verify: host BLAS results depend on the GEMM's row
    count (thread partitioning), so decode steps and windows run the same
    padded row count ``rows``, and window attention runs query row by query
    row (a batched einsum's result depends on the window length)."""

    def __init__(self, oracle: Qwen2Oracle, rows: int | None = None):
        self.o = oracle
        self.rows = rows
        self.kc: list[list[torch.Tensor]] = []
        self.vc: list[list[torch.Tensor]] = []

    @torch.no_grad()
    def forward(self, windows, prefill: bool = False) -> list[torch.Tensor]:
        """``windows`` = [(request, tokens, start)]; positions [start, start +
        len) of each request, keys [0, start) from its cache.  Returns the
        logits of each window's rows."""
        o, s = self.o, self.o.s
        nq, nkv, hd = s.q_heads, s.kv_heads, s.head_dim
        G = nq // nkv
        toks = [t for _, ts, _ in windows for t in ts]
        lens = [len(ts) for _, ts, _ in windows]
        n_real = len(toks)
        if not prefill and self.rows:
            if n_real > self.rows:
                raise ValueError("window rows exceed the port's fixed row count")
            toks += [0] * (self.rows - n_real)
        x = o.embed[torch.as_tensor(toks, dtype=torch.long)].to(o.acc)
        scale = float(np.sqrt(hd))
        for li, L in enumerate(o.layers):
            qkv = o._normed_proj(x, L["ln1"], L["wqkv"]) + L["bqkv"]
            outs, r0 = [], 0
            for (req, ts, start), T in zip(windows, lens):
                pos = torch.arange(start, start + T)
                blk = qkv[r0:r0 + T]
                r0 += T
                q = o._rope(blk[:, : nq * hd].view(T, nq, hd), pos)
                k = o._rope(blk[:, nq * hd: (nq + nkv) * hd].view(T, nkv, hd), pos)
                v = o._r(blk[:, (nq + nkv) * hd:].view(T, nkv, hd))
                kc = torch.cat([self.kc[req][li][:start], k]) if start else k
                vc = torch.cat([self.vc[req][li][:start], v]) if start else v
                self.kc[req][li], self.vc[req][li] = kc, vc
                kk, vv = kc.repeat_interleave(G, 1), vc.repeat_interleave(G, 1)
                if prefill:
                    sc = torch.einsum("qhd,khd->hqk", q, kk) / scale
                    sc = sc.masked_fill(torch.ones(T, start + T, dtype=torch.bool).triu(start + 1), float("-inf"))
                    p = torch.exp(sc - sc.amax(-1, keepdim=True))
                    l = p.sum(-1, keepdim=True)
                    outs.append(torch.einsum("hqk,khd->qhd", o._r(p), vv) / l.permute(1, 0, 2))
                    continue
                for i in range(T):   # one query row at a time: window-length invariant
                    n = start + i + 1
                    sc = torch.einsum("hd,khd->hk", q[i], kk[:n]) / scale
                    p = torch.exp(sc - sc.amax(-1, keepdim=True))
                    l = p.sum(-1, keepdim=True)
                    outs.append((torch.einsum("hk,khd->hd", o._r(p), vv[:n]) / l)[None])
            att = torch.cat(outs).reshape(-1, nq * hd)
            if att.shape[0] < x.shape[0]:
                att = torch.cat([att, att.new_zeros(x.shape[0] - att.shape[0], nq * hd)])
            x = x + o._r(att) @ L["wo"].t()
            g = o._normed_proj(x, L["ln2"], L["wg"])
            u = o._normed_proj(x, L["ln2"], L["wu"])
            x = x + o._r(g / (1.0 + torch.exp(-g)) * u) @ L["wd"].t()
        lg = o._normed_proj(x[:n_real], o.final_norm, o.lm_head)
        return list(torch.split(lg, lens))

    def prefill(self, prompts) -> None:
        """Cache every prompt token but the last (the first window starts from it)."""
        for p in prompts:
            self.kc.append([None] * len(self.o.layers))
            self.vc.append([None] * len(self.o.layers))
        self.forward([(r, list(p[:-1]), 0) for r, p in enumerate(prompts) if len(p) > 1], prefill=True)

    def greedy(self, prompts, steps: int) -> list[list[int]]:
        """Plain batched greedy decode of ``steps`` tokens per request (the
        target continuation the reference-acceptance drafter proposes)."""
        seqs = [list(p) for p in prompts]
        out = [[] for _ in prompts]
        for _ in range(steps):
            lg = self.forward([(r, [s[-1]], len(s) - 1) for r, s in enumerate(seqs)])
            for r, l in enumerate(lg):
                t = int(torch.argmax(l[-1]))
                out[r].append(t)
                seqs[r].append(t)
        return out

    def window(self, seqs, drafts, bonus: bool = True) -> list[tuple[int, int, int]]:
        """One speculation window for every request: verify ``drafts[r]``
        after ``seqs[r]`` (committed tokens, extended in place).  Returns
        per-request (proposed, accepted, committed)."""
        lg = self.forward([(r, [s[-1]] + list(d), len(s) - 1) for r, (s, d) in enumerate(zip(seqs, drafts))])
        res = []
        for r, (s, d) in enumerate(zip(seqs, drafts)):
            y = [int(t) for t in torch.argmax(lg[r], -1)]
            a = 0
            while a < len(d) and d[a] == y[a]:
                a += 1
            c = (len(d) + (1 if bonus else 0)) if (a == len(d) and d) else a + 1
            s += y[:c]
            res.append((len(d), a, c))
        return res
