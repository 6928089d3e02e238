"""Tiny HF transformers models (test infrastructure): the same shapes as the engine's tiny configs
(configs.TINY / TINY_DSV2, small vocab), random-init by HF itself, saved as safetensors checkpoints
in the Hub format HF 5.5 writes."""

from __future__ import annotations

import torch


def tiny_mixtral_hf(layers: int = 2, vocab: int = 512, seed: int = 0):
    from transformers import MixtralConfig, MixtralForCausalLM

    torch.manual_seed(seed)
    cfg = MixtralConfig(vocab_size=vocab, hidden_size=256, intermediate_size=512, num_hidden_layers=layers,
                        num_attention_heads=8, num_key_value_heads=2, head_dim=32, num_local_experts=8,
                        num_experts_per_tok=2, rope_theta=1e6, rms_norm_eps=1e-5)
    m = MixtralForCausalLM(cfg).to(torch.bfloat16).eval()
    with torch.no_grad():  # non-trivial norms, so the loader's norm mapping is exercised
        for n, p in m.named_parameters():
            if "norm" in n:
                p.copy_(1.0 + 0.1 * torch.randn_like(p.float()).to(p.dtype))
    return m


def tiny_dsv2_hf(layers: int = 3, vocab: int = 512, seed: int = 0):
    from transformers import DeepseekV2Config, DeepseekV2ForCausalLM

    torch.manual_seed(seed)
    cfg = DeepseekV2Config(vocab_size=vocab, hidden_size=256, intermediate_size=512, moe_intermediate_size=128,
                           num_hidden_layers=layers, num_attention_heads=4, num_key_value_heads=4,
                           n_routed_experts=16, n_shared_experts=2, num_experts_per_tok=4, first_k_dense_replace=1,
                           kv_lora_rank=128, q_lora_rank=None, qk_nope_head_dim=32, qk_rope_head_dim=32, v_head_dim=32,
                           topk_method="group_limited_greedy", n_group=4, topk_group=2, routed_scaling_factor=2.0,
                           rope_theta=10000.0, rms_norm_eps=1e-6)
    m = DeepseekV2ForCausalLM(cfg).to(torch.bfloat16).eval()
    with torch.no_grad():
        for n, p in m.named_parameters():
            if "norm" in n:
                p.copy_(1.0 + 0.1 * torch.randn_like(p.float()).to(p.dtype))
    # HF 5.5.0 DeepseekV2Moe.route_tokens_to_experts reads self.num_experts for group_limited_greedy
    # (modeling_deepseek_v2.py:112) but never sets it (same workaround as tests/golden/make_golden.py)
    for layer in m.model.layers:
        if hasattr(layer.mlp, "experts"):
            layer.mlp.num_experts = cfg.n_routed_experts
    return m


def save(model, path, max_shard_size=None) -> str:
    kw = {} if max_shard_size is None else {"max_shard_size": max_shard_size}
    model.save_pretrained(path, safe_serialization=True, **kw)
    return str(path)
