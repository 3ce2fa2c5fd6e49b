"""Target / drafter decoder shapes, deterministic random-init weights, and the
device-resident model (weights + paged KV cache + workspace) behind
``sr_model_*``.

The reference has no model (the target token is a keyed random
integer, ``sim.py:313-320``).  BASELINE.json names Qwen2.5-shaped targets, so
the verification forward here is a Qwen2-architecture decoder (RMSNorm,
RoPE theta 1e6, GQA with QKV bias, SwiGLU MLP) with random N(0, 0.02)
weights from a seeded generator.  The same canonical weights feed the CPU
oracle (``oracle/qwen2_oracle.py``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import ConfigError

PAGE = 64  # tokens per KV page (= attention key tile)


@dataclass(frozen=True)
class ModelShape:
    name: str
    hidden: int
    intermediate: int
    layers: int
    q_heads: int
    kv_heads: int
    head_dim: int
    vocab: int
    tied: bool
    rope_theta: float = 1e6
    rms_eps: float = 1e-6

    @property
    def qkv_width(self) -> int:
        return (self.q_heads + 2 * self.kv_heads) * self.head_dim

    def linear_params(self) -> int:
        """Parameters touched by the verify GEMMs per token (incl. lm_head)."""
        h, i = self.hidden, self.intermediate
        per_layer = h * self.qkv_width + self.q_heads * self.head_dim * h + 3 * h * i
        return self.layers * per_layer + self.vocab * h

    def kv_bytes_per_token(self, esize: int = 2) -> int:
        return self.layers * 2 * self.kv_heads * self.head_dim * esize


# Public Qwen2.5 config.json shapes; "tiny" is this repo's
# CPU-runnable config-1 target (vocab = the reference's _VOCAB, sim.py:41).
SHAPES = {
    "tiny": ModelShape("tiny", 256, 512, 2, 4, 2, 64, 50257, True),
    "qwen2.5-0.5b": ModelShape("qwen2.5-0.5b", 896, 4864, 24, 14, 2, 64, 151936, True),
    "qwen2.5-1.5b": ModelShape("qwen2.5-1.5b", 1536, 8960, 28, 12, 2, 128, 151936, True),
    "qwen2.5-7b": ModelShape("qwen2.5-7b", 3584, 18944, 28, 28, 4, 128, 152064, False),
    "qwen2.5-32b": ModelShape("qwen2.5-32b", 5120, 27648, 64, 40, 8, 128, 152064, False),
}


def shape(name: str, layers: int | None = None) -> ModelShape:
    if name not in SHAPES:
        raise ConfigError(f"unknown model shape {name!r}; known: {sorted(SHAPES)}")
    s = SHAPES[name]
    if layers is not None:
        s = ModelShape(**{**s.__dict__, "layers": layers, "name": f"{s.name}-L{layers}"})
    return s


def init_weights(s: ModelShape, seed: int = 0, device="cpu", std: float = 0.02, lazy: bool = False) -> dict:
    """Canonical (HF-layout) fp32 weights, N(0, std), deterministic in seed.

    Norm weights are 1 + N(0, std) so the scale is exercised; biases N(0, std).
    ``lazy``: ``w["layers"]`` is a one-pass iterable that creates each layer
    when reached (own generator per layer), so a model whose fp32 weights do
    not fit next to its bf16 copy (32B) converts layer by layer.
    """
    g = torch.Generator(device=device).manual_seed(seed)

    def rnd(*shape_, gen=g):
        return torch.randn(*shape_, generator=gen, device=device, dtype=torch.float32) * std

    h, i, hd = s.hidden, s.intermediate, s.head_dim

    def layer(gen):
        return {
            "ln1": 1.0 + rnd(h, gen=gen),
            "wq": rnd(s.q_heads * hd, h, gen=gen), "wk": rnd(s.kv_heads * hd, h, gen=gen),
            "wv": rnd(s.kv_heads * hd, h, gen=gen),
            "bq": rnd(s.q_heads * hd, gen=gen), "bk": rnd(s.kv_heads * hd, gen=gen),
            "bv": rnd(s.kv_heads * hd, gen=gen),
            "wo": rnd(h, s.q_heads * hd, gen=gen),
            "ln2": 1.0 + rnd(h, gen=gen),
            "wg": rnd(i, h, gen=gen), "wu": rnd(i, h, gen=gen), "wd": rnd(h, i, gen=gen),
        }

    w = {"embed": rnd(s.vocab, h)}
    if lazy:
        w["layers"] = (layer(torch.Generator(device=device).manual_seed(seed * 1000 + 1 + li))
                       for li in range(s.layers))
    else:
        w["layers"] = [layer(g) for _ in range(s.layers)]
    w["final_norm"] = 1.0 + rnd(h)
    w["lm_head"] = w["embed"] if s.tied else rnd(s.vocab, h)
    return w


def interleave_gate_up(wg: torch.Tensor, wu: torch.Tensor) -> torch.Tensor:
    """[2I, H]: per 32 rows, 16 gate rows then the matching 16 up rows (the
    SwiGLU GEMM epilogue pairs them inside one 32-column accumulator chunk)."""
    I, H = wg.shape
    return torch.stack([wg.view(I // 16, 16, H), wu.view(I // 16, 16, H)], dim=1).reshape(2 * I, H)


def pair_interleave_heads(w: torch.Tensor, heads: int, hd: int) -> torch.Tensor:
    """q/k projection rows (or bias) per head reordered (d, d + hd/2) pairwise:
    row 2i = dim i, row 2i+1 = dim i + hd/2.  The fused qkv + RoPE GEMM
    epilogue (gemm.cuh RopeArgs) then finds 16 whole rotation pairs in every
    32-column accumulator chunk."""
    half = hd // 2
    rest = tuple(w.shape[1:])
    return w.reshape(heads, 2, half, *rest).transpose(1, 2).reshape(heads * hd, *rest)


def pair_deinterleave_heads(w: torch.Tensor, heads: int, hd: int) -> torch.Tensor:
    """Inverse of :func:`pair_interleave_heads`."""
    half = hd // 2
    rest = tuple(w.shape[1:])
    return w.reshape(heads, half, 2, *rest).transpose(1, 2).reshape(heads * hd, *rest)


def qkv_rows(L: dict, s, fused_rope: bool):
    """Concatenated W_qkv [(nq + 2 nkv) hd, H] and bias in kernel row order."""
    wq, wk, bq, bk = L["wq"], L["wk"], L["bq"], L["bk"]
    if fused_rope:
        wq, bq = pair_interleave_heads(wq, s.q_heads, s.head_dim), pair_interleave_heads(bq, s.q_heads, s.head_dim)
        wk, bk = pair_interleave_heads(wk, s.kv_heads, s.head_dim), pair_interleave_heads(bk, s.kv_heads, s.head_dim)
    return torch.cat([wq, wk, L["wv"]], 0), torch.cat([bq, bk, L["bv"]], 0)


def rope_tables(s: ModelShape, max_pos: int):
    """cos/sin [max_pos, hd/2] float32 computed in float64 (shared with the oracle)."""
    half = s.head_dim // 2
    inv = s.rope_theta ** (-np.arange(half, dtype=np.float64) * 2.0 / s.head_dim)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


class DeviceModel:
    """Weights in kernel layout + paged KV cache + workspace on one GPU."""

    def __init__(self, s: ModelShape, weights: dict, *, dtype: str = "bf16", max_requests: int,
                 max_len: int, max_tokens: int, max_seqs: int, branches: int = 0,
                 window_max: int = 8, logits_capacity: int = 0, device="cuda"):
        self.lib = _native.lib()
        self.s = s
        self.dev = torch.device(device)
        self.dtype_code = 1 if dtype == "bf16" else 0
        self.tdtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        td = self.tdtype

        def put(t, as_type=None):
            return t.to(device=self.dev, dtype=as_type or td).contiguous()

        self.embed = put(weights["embed"])
        self.lm_head = self.embed if s.tied else put(weights["lm_head"])
        self.final_norm = put(weights["final_norm"], torch.float32)
        self.layer_tensors = []
        ptrs = []
        # bf16: RoPE + KV scatter run in the qkv GEMM epilogue, which wants the
        # q/k rows pair-interleaved (sr_model_desc, include/specrollout.h)
        self.fused_rope = self.dtype_code == 1
        for L in weights["layers"]:
            w_qkv, b_qkv = qkv_rows(L, s, self.fused_rope)
            t = {
                "ln1": put(L["ln1"], torch.float32),
                "w_qkv": put(w_qkv),
                "b_qkv": put(b_qkv, torch.float32),
                "w_o": put(L["wo"]),
                "ln2": put(L["ln2"], torch.float32),
                "w_gu": put(interleave_gate_up(L["wg"].to(self.dev), L["wu"].to(self.dev))),
                "w_down": put(L["wd"]),
            }
            self.layer_tensors.append(t)
            ptrs += [t[k].data_ptr() for k in ("ln1", "w_qkv", "b_qkv", "w_o", "ln2", "w_gu", "w_down")]
        self._layer_ptrs = (ctypes.c_void_p * len(ptrs))(*ptrs)

        self.max_len = max_len
        self.max_pos = max_len + 8
        cos, sin = rope_tables(s, self.max_pos)
        self.rope_cos = torch.from_numpy(cos).to(self.dev)
        self.rope_sin = torch.from_numpy(sin).to(self.dev)

        self.pages_per_req = math.ceil(max_len / PAGE)
        self.num_pages = max_requests * self.pages_per_req
        # contiguous page runs per request (the block table keeps paging explicit)
        self.block_table = torch.arange(self.num_pages, dtype=torch.int32, device=self.dev).view(
            max_requests, self.pages_per_req)
        self.kv_cache = torch.zeros((s.layers, self.num_pages, 2, s.kv_heads, PAGE, s.head_dim),
                                    dtype=td, device=self.dev)
        self.branches = branches
        self.window_max = window_max
        self.window_kv = (torch.zeros((s.layers, branches, 2, s.kv_heads, window_max, s.head_dim),
                                      dtype=td, device=self.dev) if branches else None)
        d = _native.ModelDesc()
        d.hidden, d.intermediate, d.layers = s.hidden, s.intermediate, s.layers
        d.q_heads, d.kv_heads, d.head_dim, d.vocab = s.q_heads, s.kv_heads, s.head_dim, s.vocab
        d.dtype, d.rms_eps, d.max_pos = self.dtype_code, s.rms_eps, self.max_pos
        d.num_pages, d.page_size = self.num_pages, PAGE
        d.max_requests, d.max_pages_per_req = max_requests, self.pages_per_req
        d.max_branches, d.window_max = branches, window_max
        d.max_tokens, d.max_seqs, d.max_key = max_tokens, max_seqs, max_len - 1
        d.logits_capacity = logits_capacity
        d.embed, d.lm_head = self.embed.data_ptr(), self.lm_head.data_ptr()
        d.final_norm = self.final_norm.data_ptr()
        d.layer_weights = ctypes.cast(self._layer_ptrs, ctypes.c_void_p)
        d.rope_cos, d.rope_sin = self.rope_cos.data_ptr(), self.rope_sin.data_ptr()
        d.kv_cache, d.block_table = self.kv_cache.data_ptr(), self.block_table.data_ptr()
        d.window_kv = self.window_kv.data_ptr() if self.window_kv is not None else None
        nbytes = self.lib.sr_model_workspace_bytes(ctypes.byref(d))
        if nbytes == 0:
            raise ConfigError("model descriptor rejected: " + self.lib.sr_last_error().decode())
        self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.dev)
        d.workspace, d.workspace_bytes = self.workspace.data_ptr(), int(nbytes)
        self.desc = d
        self.max_tokens, self.max_seqs = max_tokens, max_seqs
        self.group = s.q_heads // s.kv_heads
        handle = ctypes.c_void_p()
        _native.check(self.lib.sr_model_create(ctypes.byref(d), ctypes.byref(handle)), "sr_model_create")
        self.handle = handle

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.sr_model_destroy(h)
            except Exception:
                pass

    def forward(self, token_ids, positions, seqs, *, num_seqs: int, max_q_len: int, max_key: int,
                out, output: int = 0, logit_rows=None, out_val=None, stream=None,
                temperature: float = 0.0, seed: int = 0, live_rows=None) -> None:
        """Enqueue one forward (``output`` 0 = argmax ids, 1 = fp32 logits,
        2 = keyed Gumbel-max sample at ``temperature``)."""
        a = _native.ForwardArgs()
        a.num_tokens = token_ids.numel()
        a.num_seqs = num_seqs
        a.max_q_len, a.max_key, a.output = max_q_len, max_key, output
        a.num_logit_rows = logit_rows.numel() if logit_rows is not None else 0
        a.token_ids, a.positions, a.seqs = token_ids.data_ptr(), positions.data_ptr(), seqs.data_ptr()
        a.logit_rows = logit_rows.data_ptr() if logit_rows is not None else None
        a.out = out.data_ptr()
        a.out_val = out_val.data_ptr() if out_val is not None else None
        a.temperature, a.seed = float(temperature), int(seed) & 0xFFFFFFFF
        a.live_rows = live_rows.data_ptr() if live_rows is not None else None
        _native.check(self.lib.sr_model_forward(self.handle, ctypes.byref(a),
                                                _native.stream_handle(stream)), "sr_model_forward")

    def max_prefill_seqs(self, q_len: int) -> int:
        """How many q_len-token sequences one forward can attend for."""
        budget = self.max_seqs + (self.max_tokens * self.group + 31) // 32
        return max(1, budget // max(1, math.ceil(q_len * self.group / 32)))


def seq_table(rows: list[tuple[int, int, int, int, int]], device) -> torch.Tensor:
    """SeqInfo[] from (q_start, q_len, request, ctx_len, branch) tuples."""
    arr = np.zeros((max(len(rows), 1), 8), dtype=np.int32)
    for i, r in enumerate(rows):
        arr[i, :5] = r
    return torch.from_numpy(arr).to(device)
