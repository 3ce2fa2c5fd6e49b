"""CPU: pin the model oracle.  The reference has no model, so the PyTorch-CPU
restatement (oracle/qwen2_oracle.py) is cross-checked against an independent
implementation of the same architecture -- transformers' Qwen2ForCausalLM --
on identical random-init weights; plus host-side model utilities."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle.qwen2_oracle import Qwen2Oracle


def hf_model(s, w):
    from transformers import Qwen2Config, Qwen2ForCausalLM

    cfg = Qwen2Config(vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.intermediate,
                      num_hidden_layers=s.layers, num_attention_heads=s.q_heads,
                      num_key_value_heads=s.kv_heads, head_dim=s.head_dim, rms_norm_eps=s.rms_eps,
                      tie_word_embeddings=s.tied, max_position_embeddings=4096,
                      rope_parameters={"rope_type": "default", "rope_theta": s.rope_theta})
    cfg._attn_implementation = "eager"
    m = Qwen2ForCausalLM(cfg).double().eval()
    sd = {"model.embed_tokens.weight": w["embed"], "model.norm.weight": w["final_norm"],
          "lm_head.weight": w["lm_head"]}
    for i, L in enumerate(w["layers"]):
        p = f"model.layers.{i}."
        sd.update({
            p + "input_layernorm.weight": L["ln1"], p + "post_attention_layernorm.weight": L["ln2"],
            p + "self_attn.q_proj.weight": L["wq"], p + "self_attn.q_proj.bias": L["bq"],
            p + "self_attn.k_proj.weight": L["wk"], p + "self_attn.k_proj.bias": L["bk"],
            p + "self_attn.v_proj.weight": L["wv"], p + "self_attn.v_proj.bias": L["bv"],
            p + "self_attn.o_proj.weight": L["wo"], p + "mlp.gate_proj.weight": L["wg"],
            p + "mlp.up_proj.weight": L["wu"], p + "mlp.down_proj.weight": L["wd"],
        })
    m.load_state_dict({k: v.double() for k, v in sd.items()}, strict=False)
    return m


def test_oracle_fp32_matches_transformers_qwen2():
    from paper_2511_16193_b200.model import init_weights, shape

    s = shape("tiny")
    w = init_weights(s, seed=0)
    ora = Qwen2Oracle(s, w, "fp32")
    hf = hf_model(s, w)
    toks = np.random.default_rng(0).integers(0, s.vocab, size=57).tolist()
    with torch.no_grad():
        exp = hf(torch.tensor([toks])).logits[0]
    got = ora.logits(toks)
    err = float((got - exp).abs().max() / exp.abs().max())
    assert err < 1e-6, err


def test_oracle_bf16_close_to_fp32():
    from paper_2511_16193_b200.model import init_weights, shape

    s = shape("tiny")
    w = init_weights(s, seed=1)
    toks = list(range(100, 160))
    a = Qwen2Oracle(s, w, "fp32").logits(toks)
    b = Qwen2Oracle(s, w, "bf16").logits(toks)
    assert float((a - b.double()).abs().max() / a.abs().max()) < 3e-2


def test_interleave_gate_up_layout():
    from paper_2511_16193_b200.model import interleave_gate_up

    g = torch.arange(32 * 3).view(32, 3).float()
    u = -g
    w = interleave_gate_up(g, u)
    assert torch.equal(w[:16], g[:16]) and torch.equal(w[16:32], u[:16])
    assert torch.equal(w[32:48], g[16:32]) and torch.equal(w[48:64], u[16:32])


def test_pair_interleave_heads_layout():
    from paper_2511_16193_b200.model import pair_deinterleave_heads, pair_interleave_heads

    w = torch.arange(2 * 8 * 3).view(16, 3).float()   # 2 heads, hd 8
    p = pair_interleave_heads(w, 2, 8)
    # head 0: rows 0,4,1,5,2,6,3,7; head 1 the same + 8
    order = [0, 4, 1, 5, 2, 6, 3, 7]
    assert torch.equal(p[:8], w[order]) and torch.equal(p[8:], w[[8 + i for i in order]])
    assert torch.equal(pair_deinterleave_heads(p, 2, 8), w)
    b = torch.arange(16).float()
    assert torch.equal(pair_deinterleave_heads(pair_interleave_heads(b, 2, 8), 2, 8), b)


def test_shapes_and_roofline_params():
    from paper_2511_16193_b200.model import SHAPES

    # SURVEY §8d P_lin figures (linear params incl. lm_head)
    assert abs(SHAPES["qwen2.5-1.5b"].linear_params() / 1.544e9 - 1) < 0.01
    assert abs(SHAPES["qwen2.5-7b"].linear_params() / 7.070e9 - 1) < 0.01
    assert abs(SHAPES["qwen2.5-32b"].linear_params() / 31.98e9 - 1) < 0.01
    assert SHAPES["qwen2.5-1.5b"].kv_bytes_per_token() == 28672
    assert SHAPES["qwen2.5-7b"].kv_bytes_per_token() == 57344


def test_batched_rollout_port_matches_oracle():
    """The batched CPU port timed by bench.py's reference arm: its greedy
    continuation equals the oracle's, and speculation windows with wrong
    drafts still commit exactly that continuation."""
    import numpy as np

    from oracle.qwen2_oracle import BatchedRollout, Qwen2Oracle
    from paper_2511_16193_b200.model import init_weights, shape

    s = shape("tiny")
    o = Qwen2Oracle(s, init_weights(s, seed=0), "bf16")
    rng = np.random.default_rng(1)
    ps = [rng.integers(0, s.vocab, int(rng.integers(5, 30))).tolist() for _ in range(3)]
    port = BatchedRollout(o, rows=3 * 4)
    port.prefill(ps)
    g = port.greedy(ps, 10)
    assert g == [o.greedy(p, 10) for p in ps]
    seqs, gen = [list(p) for p in ps], [0, 0, 0]
    while min(gen) < 10:
        d = [[g[r][gen[r] + j] if j != 2 else (g[r][gen[r] + j] + 1) % s.vocab
              for j in range(3) if gen[r] + j < 10] for r in range(3)]
        for r, (n, a, c) in enumerate(port.window(seqs, d)):
            assert a == min(n, 2)
            gen[r] += c
    assert all(seqs[r][len(ps[r]):][:10] == g[r] for r in range(3))
