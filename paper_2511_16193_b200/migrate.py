"""Request migration between rollout engines (straggler pull / tail
rebalancing as real data movement; reference ``sim.py:546-625``
``pull_straggler`` / ``_rebalance_tail`` and the ``scale_charge`` cost model
``bon.py:65-72``, ``scenarios.py:84-88``, which the reference prices at 50 ms
+ 0.01 ms/token).

A request's state is its token row, its lengths and budget, and the KV of
every committed position but the last (the engine invariant) in each layer.
The paged cache keeps a request's pages in its block-table row, so the KV
moves as whole 64-token pages in the cache's native layout (bf16 pages keep
their slot swizzle: same slot, same bytes).  Locally the copy is a device /
peer copy; across ranks it is one batched NCCL send/recv over NVLink.
"""

from __future__ import annotations

import math

import torch

from .errors import ConfigError

PAGE = 64


def _pages(eng, b: int) -> int:
    kv_len = int(eng.seq_len[b]) - 1
    return max(0, math.ceil(kv_len / PAGE))


def _check_compatible(src, dst) -> None:
    a, b = src.m, dst.m
    if (a.s.layers, a.s.kv_heads, a.s.head_dim, a.dtype_code) != (b.s.layers, b.s.kv_heads, b.s.head_dim,
                                                                   b.dtype_code):
        raise ConfigError("migration needs engines over the same model shape and dtype")
    if src.k != dst.k:
        raise ConfigError("migration needs the same window k")


def _synthetic(eng) -> list:
    from .engine import SyntheticDrafter

    return [d for d in eng.drafters if isinstance(d, SyntheticDrafter)]


def pack_request(eng, b: int) -> dict:
    """Gather request ``b``'s state into contiguous device tensors.  A
    reference-acceptance (synthetic) drafter's per-slot rows -- the request's
    target continuation, its keyed accept uniforms and latent rate -- travel
    with it, so the request keeps drafting under the same law."""
    n = _pages(eng, b)
    pages = eng.m.block_table[b, :n].long()
    L = int(eng.seq_len[b])
    st = {
        "lens": torch.stack([eng.seq_len[b], eng.gen_len[b], eng.max_new[b],
                             torch.tensor(n, dtype=torch.int32, device=eng.dev)]).to(torch.int32),
        "tokens": eng.tokens[b, :L].clone(),
        "kv": eng.m.kv_cache[:, pages].contiguous(),   # [layers, n, 2, kv_heads, 64, hd]
    }
    for i, d in enumerate(_synthetic(eng)):
        st[f"syn{i}_truth"] = d.truth[b].clone()
        st[f"syn{i}_u"] = d.uniforms[b].clone()
        st[f"syn{i}_meta"] = torch.stack([d.p[b], d.truth_len[b].to(torch.float64)])
    return st


def _check_room(eng, seq_len: int, gen_len: int, max_new: int, n: int) -> None:
    """The destination slot must hold the request to its END, not just its
    current length: its remaining budget is written into the token row and
    the KV pages, and attention runs with the engine's ``max_key``."""
    final = seq_len + max(0, max_new - gen_len)
    if final + eng.k + 2 > min(eng.stride, eng.max_key + 1) or n > eng.m.pages_per_req:
        raise ConfigError(f"destination engine sized for {min(eng.stride, eng.max_key + 1)} positions per "
                          f"request; the migrated request needs {final + eng.k + 2}")


def unpack_request(eng, b: int, st: dict) -> None:
    """Install a packed request into slot ``b`` of ``eng`` (same model shape).

    Host and drafter state of the slot follow the new occupant: the prompt
    length (``outputs()`` slices at it), the slot capacity, and a model
    drafter's cache (re-prefilled from the token row).  A synthetic drafter
    proposes from a per-slot truth row of the previous occupant, so slots of
    such engines cannot take migrated requests."""
    from .engine import ModelDrafter, SyntheticDrafter

    seq_len, gen_len, max_new, n = (int(x) for x in st["lens"].tolist())
    _check_room(eng, seq_len, gen_len, max_new, n)
    syn = _synthetic(eng)
    for i, d in enumerate(syn):
        if f"syn{i}_truth" not in st:
            raise ConfigError("engines with a synthetic drafter hold per-slot truth rows; the migrated "
                              "request must bring its own (from an engine with the same drafters)")
        if st[f"syn{i}_truth"].numel() > d.truth.shape[1]:
            raise ConfigError("destination synthetic drafter rows are shorter than the request's")
    eng.tokens[b, :seq_len].copy_(st["tokens"][:seq_len])
    eng.seq_len[b] = seq_len
    eng.gen_len[b] = gen_len
    eng.max_new[b] = max_new
    eng.max_new_cap[b] = max_new
    eng.prompt_lens[b] = seq_len - gen_len
    if n:
        pages = eng.m.block_table[b, :n].long()
        eng.m.kv_cache[:, pages] = st["kv"][:, :n].to(eng.m.kv_cache.device)
    for d in eng.drafters:
        if isinstance(d, ModelDrafter) and d.eng is eng:
            d.reset_slot(b)
    for i, d in enumerate(syn):
        t, u = st[f"syn{i}_truth"], st[f"syn{i}_u"]
        d.truth[b].zero_()
        d.truth[b, : t.numel()].copy_(t)
        d.uniforms[b].zero_()
        d.uniforms[b, : u.numel()].copy_(u)
        meta = st[f"syn{i}_meta"].to(d.p.device)
        d.p[b] = meta[0]
        d.truth_len[b] = meta[1].to(torch.int32)


def migrate_local(src, b_src: int, dst, b_dst: int) -> int:
    """Move request ``b_src`` of ``src`` into slot ``b_dst`` of ``dst`` (same
    or peer GPU); the source slot is retired (budget exhausted).  Returns the
    bytes moved."""
    _check_compatible(src, dst)
    st = pack_request(src, b_src)
    if src.dev != dst.dev:
        st = {k: v.to(dst.dev, non_blocking=True) for k, v in st.items()}
    unpack_request(dst, b_dst, st)
    src.retire(b_src)
    return sum(v.numel() * v.element_size() for v in st.values())


def _host_staged(dist) -> bool:
    """gloo (CPU tests, one-GPU multi-process runs) moves host tensors only."""
    return dist.get_backend() == "gloo"


def _p2p(dist, kind: str, tensors: list, peer: int) -> None:
    """Post one batch of sends or receives to ``peer`` and wait for it."""
    fn = dist.isend if kind == "send" else dist.irecv
    ops = [dist.P2POp(fn, t, peer) for t in tensors if t.numel()]
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def send_requests(dist, eng, bs: list[int], peer: int) -> int:
    """P2P (NCCL over NVLink, or host-staged gloo): ship requests ``bs`` to
    rank ``peer`` (which calls :func:`recv_requests` with the same count) as
    a meta table, then all token rows, all KV pages and any synthetic drafter
    rows in one batch; retire them here.  Returns the bytes sent."""
    sts = [pack_request(eng, b) for b in bs]
    meta = torch.stack([st["lens"] for st in sts])
    payload = [torch.cat([st["tokens"] for st in sts]), torch.cat([st["kv"] for st in sts], 1).contiguous()]
    for i in range(len(_synthetic(eng))):
        for key in ("truth", "u", "meta"):
            payload.append(torch.stack([st[f"syn{i}_{key}"] for st in sts]).contiguous())
    if _host_staged(dist):
        meta, payload = meta.cpu(), [t.cpu() for t in payload]
    dist.send(meta, peer)
    _p2p(dist, "send", payload, peer)
    for b in bs:
        eng.retire(b)
    return meta.numel() * 4 + sum(t.numel() * t.element_size() for t in payload)


def recv_requests(dist, eng, bs: list[int], peer: int) -> None:
    """P2P: receive ``len(bs)`` requests from rank ``peer`` into slots ``bs``."""
    m = eng.m
    dev = "cpu" if _host_staged(dist) else eng.dev
    meta = torch.empty((len(bs), 4), dtype=torch.int32, device=dev)
    dist.recv(meta, peer)
    lens = meta.tolist()
    toks = torch.empty(sum(r[0] for r in lens), dtype=torch.int32, device=dev)
    npages = sum(r[3] for r in lens)
    kv = torch.empty((m.s.layers, npages) + tuple(m.kv_cache.shape[2:]), dtype=m.kv_cache.dtype, device=dev)
    payload = [toks, kv]
    syn = _synthetic(eng)
    for d in syn:
        payload += [torch.empty((len(bs), d.truth.shape[1]), dtype=torch.int32, device=dev),
                    torch.empty((len(bs), d.uniforms.shape[1]), dtype=torch.float64, device=dev),
                    torch.empty((len(bs), 2), dtype=torch.float64, device=dev)]
    _p2p(dist, "recv", payload, peer)
    payload = [t.to(eng.dev) for t in payload]
    meta = meta.to(eng.dev)
    toks, kv = payload[0], payload[1]
    t0 = p0 = 0
    for i, b in enumerate(bs):
        seq_len, n = lens[i][0], lens[i][3]
        st = {"lens": meta[i], "tokens": toks[t0:t0 + seq_len], "kv": kv[:, p0:p0 + n]}
        for j in range(len(syn)):
            st[f"syn{j}_truth"], st[f"syn{j}_u"], st[f"syn{j}_meta"] = (payload[2 + 3 * j][i], payload[3 + 3 * j][i],
                                                                         payload[4 + 3 * j][i])
        unpack_request(eng, b, st)
        t0 += seq_len
        p0 += n
