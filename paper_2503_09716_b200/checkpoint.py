"""On-disk weights: HuggingFace safetensors checkpoints of the two model families the engine runs.

The paper's engine runs real HF checkpoints (reference PAPER.md:696); the reference's memory model
stages every expert as one contiguous `expert_bytes` blob and every layer's dense modules as one
blob (offload_dag.py:308-321, 438-445).  This module reads a checkpoint directory (config.json +
model.safetensors or a sharded model.safetensors.index.json, memory-mapped by `safetensors`) and
hands out each layer in the engine's layout:

  Mixtral   q/k/v_proj -> wqkv [(Hq + 2 Hkv) hd, d] (rows q | k | v); o_proj -> wo;
            block_sparse_moe.experts.{e}.w1 / w3 / w2 (gate / up / down, the Hub format HF 5.5
            writes) or the fused mlp.experts.gate_up_proj / down_proj -> w_gate_up [E, 2f, d]
            (gate rows then up rows, MixtralExperts, modeling_mixtral.py:70-71), w_down [E, d, f];
            gate -> router [E, d]; input / post_attention_layernorm -> ln1 / ln2.
  DeepSeek  q_proj or q_a_proj + q_a_layernorm + q_b_proj; kv_a_proj_with_mqa, kv_a_layernorm,
  -V2       kv_b_proj, o_proj (modeling_deepseek_v2.py:337-396); mlp.experts.{e}.gate / up /
            down_proj -> w_gate_up / w_down as above; mlp.shared_experts.* -> sh_gate_up [1, 2 fs, d]
            / sh_down [1, d, fs]; the first_k_dense_replace layers' mlp.gate / up / down_proj ->
            dense_gate_up / dense_down.

Tensors are converted to bf16 on load (the engine computes in bf16).  The engine then either keeps
them in HBM or packs the uncached ones into pinned expert-contiguous host blobs, one DMA per expert
copy (offload.py).  Only default RoPE is implemented: a checkpoint with rope scaling (e.g. YaRN) is
refused rather than run with the wrong positions.
"""

from __future__ import annotations

import json
import os
from dataclasses import replace
from typing import Any, Mapping

import torch

from .configs import ModelArch

BF16 = torch.bfloat16


def _rope_theta(cfg: Mapping[str, Any]) -> float:
    rp = cfg.get("rope_parameters") or {}
    scaling = cfg.get("rope_scaling") or {}
    kind = rp.get("rope_type", scaling.get("type", scaling.get("rope_type", "default"))) or "default"
    if kind != "default":
        raise NotImplementedError(f"rope type {kind!r} is not implemented by the engine (default RoPE only)")
    return float(rp.get("rope_theta", cfg.get("rope_theta", 10000.0)))


def arch_from_hf_config(cfg: Mapping[str, Any], name: str | None = None) -> ModelArch:
    """ModelArch of an HF config.json (model_type "mixtral" or "deepseek_v2")."""
    mt = cfg.get("model_type")
    if mt == "mixtral":
        hd = cfg.get("head_dim") or cfg["hidden_size"] // cfg["num_attention_heads"]
        return ModelArch(name=name or "mixtral-checkpoint", family="mixtral", vocab=cfg["vocab_size"],
                         hidden=cfg["hidden_size"], layers=cfg["num_hidden_layers"],
                         n_heads=cfg["num_attention_heads"], n_kv_heads=cfg["num_key_value_heads"], head_dim=hd,
                         moe_ffn=cfg["intermediate_size"], n_experts=cfg["num_local_experts"],
                         top_k=cfg["num_experts_per_tok"], rope_theta=_rope_theta(cfg), rms_eps=cfg["rms_norm_eps"])
    if mt == "deepseek_v2":
        method = cfg.get("topk_method", "greedy")
        if method not in ("greedy", "group_limited_greedy"):
            raise NotImplementedError(f"topk_method {method!r}")
        if cfg.get("norm_topk_prob", False):
            raise NotImplementedError("norm_topk_prob=True")
        nope, rope = cfg["qk_nope_head_dim"], cfg["qk_rope_head_dim"]
        return ModelArch(name=name or "deepseek-v2-checkpoint", family="deepseek_v2", vocab=cfg["vocab_size"],
                         hidden=cfg["hidden_size"], layers=cfg["num_hidden_layers"],
                         n_heads=cfg["num_attention_heads"], n_kv_heads=cfg["num_attention_heads"],
                         head_dim=nope + rope, moe_ffn=cfg["moe_intermediate_size"], n_experts=cfg["n_routed_experts"],
                         top_k=cfg["num_experts_per_tok"], rope_theta=_rope_theta(cfg), rms_eps=cfg["rms_norm_eps"],
                         n_shared=cfg.get("n_shared_experts") or 0, first_k_dense=cfg.get("first_k_dense_replace", 0),
                         dense_ffn=cfg["intermediate_size"], q_lora_rank=cfg.get("q_lora_rank") or 0,
                         kv_lora_rank=cfg["kv_lora_rank"], qk_nope_dim=nope, qk_rope_dim=rope,
                         v_head_dim=cfg["v_head_dim"], routed_scaling=float(cfg.get("routed_scaling_factor", 1.0)),
                         topk_method=method, n_group=cfg.get("n_group") or 1, topk_group=cfg.get("topk_group") or 1)
    raise NotImplementedError(f"model_type {mt!r}: the engine runs the mixtral and deepseek_v2 families")


class Checkpoint:
    """A HF safetensors checkpoint directory, read lazily (memory-mapped)."""

    def __init__(self, path: str, layers: int | None = None):
        from safetensors import safe_open

        self.path = path
        with open(os.path.join(path, "config.json")) as f:
            self.config = json.load(f)
        arch = arch_from_hf_config(self.config, name=os.path.basename(os.path.normpath(path)))
        self.arch = replace(arch, layers=layers) if layers is not None else arch
        idx = os.path.join(path, "model.safetensors.index.json")
        if os.path.exists(idx):
            with open(idx) as f:
                weight_map = json.load(f)["weight_map"]
        else:
            single = os.path.join(path, "model.safetensors")
            if not os.path.exists(single):
                raise FileNotFoundError(f"{path}: no model.safetensors or model.safetensors.index.json")
            from safetensors import safe_open as _so
            with _so(single, "pt") as f:
                weight_map = {k: "model.safetensors" for k in f.keys()}
        self._file_of = weight_map
        self._handles = {fn: safe_open(os.path.join(path, fn), "pt") for fn in sorted(set(weight_map.values()))}

    def has(self, name: str) -> bool:
        return name in self._file_of

    def get(self, name: str) -> torch.Tensor:
        """One tensor as bf16 on the CPU."""
        try:
            fn = self._file_of[name]
        except KeyError:
            raise KeyError(f"{self.path}: checkpoint has no tensor {name!r}") from None
        return self._handles[fn].get_tensor(name).to(BF16)

    # ---- global tensors ---------------------------------------------------------------------
    def embed(self) -> torch.Tensor:
        return self.get("model.embed_tokens.weight")

    def final_norm(self) -> torch.Tensor:
        return self.get("model.norm.weight")

    def lm_head(self) -> torch.Tensor:
        if self.has("lm_head.weight"):
            return self.get("lm_head.weight")
        return self.embed()  # tied embeddings

    # ---- per layer, engine layout -------------------------------------------------------------
    def _experts(self, p: str, n: int, names: tuple[str, str, str]) -> tuple[torch.Tensor, torch.Tensor]:
        """[n, 2f, d] gate|up and [n, d, f] down of the routed experts under prefix p."""
        g, u, dn = names
        gu = torch.stack([torch.cat([self.get(f"{p}.{e}.{g}.weight"), self.get(f"{p}.{e}.{u}.weight")], 0)
                          for e in range(n)])
        down = torch.stack([self.get(f"{p}.{e}.{dn}.weight") for e in range(n)])
        return gu, down

    def layer(self, l: int) -> dict:
        a = self.arch
        p = f"model.layers.{l}"
        L = dict(ln1=self.get(f"{p}.input_layernorm.weight"), ln2=self.get(f"{p}.post_attention_layernorm.weight"))
        if a.family == "mixtral":
            at = f"{p}.self_attn"
            L["wqkv"] = torch.cat([self.get(f"{at}.q_proj.weight"), self.get(f"{at}.k_proj.weight"),
                                   self.get(f"{at}.v_proj.weight")], 0)
            L["wo"] = self.get(f"{at}.o_proj.weight")
            if self.has(f"{p}.mlp.experts.gate_up_proj"):  # fused in-memory naming
                L["router"] = self.get(f"{p}.mlp.gate.weight")
                L["w_gate_up"] = self.get(f"{p}.mlp.experts.gate_up_proj")
                L["w_down"] = self.get(f"{p}.mlp.experts.down_proj")
            else:                                          # Hub format (w1 gate, w3 up, w2 down)
                L["router"] = self.get(f"{p}.block_sparse_moe.gate.weight")
                L["w_gate_up"], L["w_down"] = self._experts(f"{p}.block_sparse_moe.experts", a.n_experts,
                                                            ("w1", "w3", "w2"))
            return L
        at = f"{p}.self_attn"
        if a.q_lora_rank:
            L.update(q_a=self.get(f"{at}.q_a_proj.weight"), q_a_norm=self.get(f"{at}.q_a_layernorm.weight"),
                     q_b=self.get(f"{at}.q_b_proj.weight"))
        else:
            L["q_proj"] = self.get(f"{at}.q_proj.weight")
        L.update(kv_a=self.get(f"{at}.kv_a_proj_with_mqa.weight"), kv_a_norm=self.get(f"{at}.kv_a_layernorm.weight"),
                 kv_b=self.get(f"{at}.kv_b_proj.weight"), wo=self.get(f"{at}.o_proj.weight"))
        m = f"{p}.mlp"
        if l < a.first_k_dense:
            L["dense_gate_up"] = torch.cat([self.get(f"{m}.gate_proj.weight"), self.get(f"{m}.up_proj.weight")], 0)[None]
            L["dense_down"] = self.get(f"{m}.down_proj.weight")[None]
            return L
        L["router"] = self.get(f"{m}.gate.weight")
        if self.has(f"{m}.experts.gate_up_proj"):
            L["w_gate_up"], L["w_down"] = self.get(f"{m}.experts.gate_up_proj"), self.get(f"{m}.experts.down_proj")
        else:
            L["w_gate_up"], L["w_down"] = self._experts(f"{m}.experts", a.n_experts, ("gate_proj", "up_proj", "down_proj"))
        s = f"{m}.shared_experts"
        L["sh_gate_up"] = torch.cat([self.get(f"{s}.gate_proj.weight"), self.get(f"{s}.up_proj.weight")], 0)[None]
        L["sh_down"] = self.get(f"{s}.down_proj.weight")[None]
        return L


def open_checkpoint(path_or_ckpt, layers: int | None = None) -> Checkpoint:
    return path_or_ckpt if isinstance(path_or_ckpt, Checkpoint) else Checkpoint(path_or_ckpt, layers)
