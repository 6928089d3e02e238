"""On-disk weights: HF safetensors checkpoints -> the engine's layout, on the CPU
(no engine needed).  The GPU half (an engine loaded from a checkpoint vs HF itself) is
tests/test_checkpoint_gpu.py."""

import json
import os

import pytest
import torch

import hf_models
from paper_2503_09716_b200.checkpoint import Checkpoint, arch_from_hf_config


@pytest.mark.parametrize("shard", [None, "300KB"])
def test_mixtral_checkpoint_layout(tmp_path, shard):
    m = hf_models.tiny_mixtral_hf()
    path = hf_models.save(m, tmp_path / "mx", shard)
    if shard:
        assert os.path.exists(os.path.join(path, "model.safetensors.index.json"))
    ck = Checkpoint(path)
    a = ck.arch
    assert (a.family, a.hidden, a.layers, a.n_heads, a.n_kv_heads, a.head_dim, a.moe_ffn, a.n_experts, a.top_k) == \
        ("mixtral", 256, 2, 8, 2, 32, 512, 8, 2)
    assert a.rope_theta == 1e6
    sd = m.state_dict()  # HF 5.5 in-memory layout: fused experts, gate rows first
    for l in range(a.layers):
        L = ck.layer(l)
        p = f"model.layers.{l}"
        assert torch.equal(L["wqkv"], torch.cat([sd[f"{p}.self_attn.{n}_proj.weight"] for n in "qkv"], 0))
        assert torch.equal(L["w_gate_up"], sd[f"{p}.mlp.experts.gate_up_proj"])
        assert torch.equal(L["w_down"], sd[f"{p}.mlp.experts.down_proj"])
        assert torch.equal(L["router"], sd[f"{p}.mlp.gate.weight"])
        assert torch.equal(L["ln2"], sd[f"{p}.post_attention_layernorm.weight"])
    assert torch.equal(ck.lm_head(), sd["lm_head.weight"]) and torch.equal(ck.final_norm(), sd["model.norm.weight"])


def test_deepseek_checkpoint_layout(tmp_path):
    m = hf_models.tiny_dsv2_hf()
    ck = Checkpoint(hf_models.save(m, tmp_path / "ds"))
    a = ck.arch
    assert (a.family, a.first_k_dense, a.n_shared, a.kv_lora_rank, a.qk_nope_dim, a.qk_rope_dim, a.head_dim) == \
        ("deepseek_v2", 1, 2, 128, 32, 32, 64)
    assert (a.router_mode, a.n_group, a.topk_group, a.routed_scaling) == (2, 4, 2, 2.0)
    sd = m.state_dict()
    L0, L1 = ck.layer(0), ck.layer(1)
    assert torch.equal(L0["dense_gate_up"][0], torch.cat([sd["model.layers.0.mlp.gate_proj.weight"],
                                                          sd["model.layers.0.mlp.up_proj.weight"]], 0))
    assert torch.equal(L1["w_gate_up"], sd["model.layers.1.mlp.experts.gate_up_proj"])
    assert torch.equal(L1["w_down"], sd["model.layers.1.mlp.experts.down_proj"])
    assert torch.equal(L1["sh_down"][0], sd["model.layers.1.mlp.shared_experts.down_proj.weight"])
    assert torch.equal(L1["kv_b"], sd["model.layers.1.self_attn.kv_b_proj.weight"])
    assert torch.equal(L1["kv_a_norm"], sd["model.layers.1.self_attn.kv_a_layernorm.weight"])


def test_unsupported_configs_are_refused():
    base = json.loads(json.dumps({"model_type": "mixtral", "vocab_size": 8, "hidden_size": 64, "num_hidden_layers": 1,
                                  "num_attention_heads": 2, "num_key_value_heads": 1, "intermediate_size": 64,
                                  "num_local_experts": 2, "num_experts_per_tok": 1, "rms_norm_eps": 1e-5,
                                  "rope_parameters": {"rope_type": "yarn", "rope_theta": 1e4, "factor": 4.0}}))
    with pytest.raises(NotImplementedError):
        arch_from_hf_config(base)
    base["rope_parameters"] = {"rope_type": "default", "rope_theta": 1e4}
    assert arch_from_hf_config(base).rope_theta == 1e4
    with pytest.raises(NotImplementedError):
        arch_from_hf_config({"model_type": "llama"})
