"""Model architectures the engine runs (BASELINE.json configs[0..4]).

Each architecture also renders the reference planner's ModelSpec document
(reference: pkg/src/moe_planner/model_catalog.py:55-149 fields, :212-295 formulas) so the
scheduler sizes buffers and builds the job list exactly as the reference would.

Architecture constants are public HF config values (external to the reference); the tiny model
is the builder's choice pinned here.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, field, replace
from typing import Any

BYTES = 2  # bf16 everywhere


@dataclass(frozen=True)
class ModelArch:
    name: str
    family: str  # "mixtral" | "deepseek_v2"
    vocab: int
    hidden: int
    layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    moe_ffn: int  # routed expert intermediate size
    n_experts: int
    top_k: int
    rope_theta: float = 1e6
    rms_eps: float = 1e-5
    # DeepSeek-V2 extras
    n_shared: int = 0
    first_k_dense: int = 0
    dense_ffn: int = 0
    q_lora_rank: int = 0  # 0 = no q compression
    kv_lora_rank: int = 0
    qk_nope_dim: int = 0
    qk_rope_dim: int = 0
    v_head_dim: int = 0
    routed_scaling: float = 1.0
    topk_method: str = "softmax_renorm"  # mixtral | "greedy" | "group_limited_greedy"
    n_group: int = 1
    topk_group: int = 1
    init_std: float = 0.02
    extra: dict = field(default_factory=dict)

    # ---- derived ---------------------------------------------------------------------
    @property
    def is_mla(self) -> bool:
        return self.family == "deepseek_v2"

    @property
    def router_mode(self) -> int:
        return {"softmax_renorm": 0, "greedy": 1, "group_limited_greedy": 2}[self.topk_method]

    @property
    def kv_bytes_per_token_layer(self) -> int:
        if self.is_mla:
            return (self.kv_lora_rank + self.qk_rope_dim) * BYTES
        return 2 * self.n_kv_heads * self.head_dim * BYTES

    @property
    def expert_bytes(self) -> int:
        return 3 * self.hidden * self.moe_ffn * BYTES

    def attention_params(self) -> int:
        d = self.hidden
        if self.is_mla:
            H = self.n_heads
            qk = self.qk_nope_dim + self.qk_rope_dim
            q = (d * self.q_lora_rank + self.q_lora_rank * H * qk) if self.q_lora_rank else d * H * qk
            return (q + d * (self.kv_lora_rank + self.qk_rope_dim)
                    + self.kv_lora_rank * H * (self.qk_nope_dim + self.v_head_dim)
                    + H * self.v_head_dim * d)
        qd = self.n_heads * self.head_dim
        kvd = self.n_kv_heads * self.head_dim
        return d * qd + 2 * d * kvd + qd * d

    def total_params(self) -> int:
        d = self.hidden
        per_layer = self.attention_params() + 2 * d + d * self.n_experts  # norms + gate
        moe_layers = self.layers - self.first_k_dense
        p = self.layers * per_layer
        p += moe_layers * (self.n_experts * 3 * d * self.moe_ffn + self.n_shared * 3 * d * self.moe_ffn)
        p += self.first_k_dense * 3 * d * self.dense_ffn
        p += 2 * self.vocab * d + d
        return p

    def model_spec_document(self) -> dict[str, Any]:
        """The reference planner's ModelSpec document for this architecture
        (field meaning: model_catalog.py:55-88; Mixtral formula :212-239, MLA formula :242-295).
        The reference models every layer as MoE; so does this document."""
        attn = self.attention_params()
        d = self.hidden
        doc: dict[str, Any] = {
            "name": self.name,
            "num_layers": self.layers,
            "experts_per_layer": self.n_experts,
            "top_k": self.top_k,
            "shared_expert_bytes": self.n_shared * 3 * d * self.moe_ffn * BYTES,
            "attention_weights_bytes": attn * BYTES,
            "expert_bytes": self.expert_bytes,
            "kv_bytes_per_token_layer": self.kv_bytes_per_token_layer,
            "hidden_bytes_per_token": d * BYTES,
            "attn_flops_base": float(2 * attn),
            "expert_flops_per_token": float(2 * 3 * d * self.moe_ffn),
        }
        if self.is_mla:
            H = self.n_heads
            doc["attn_flops_per_context"] = float(
                2 * self.kv_lora_rank * H * self.qk_nope_dim + 2 * self.kv_lora_rank * H * self.v_head_dim
                + 2 * H * (self.qk_nope_dim + self.qk_rope_dim) + 2 * H * self.v_head_dim)
            # The reference's DSV2 preset charges the up-projected per-head K/V working set
            # (6 x H x 320 x 2 B per context token, model_catalog.py:248-254).  This engine runs
            # absorbed MLA (attn_mla.cu) straight off the 576-wide latent cache, so no per-context
            # activation exists and the term is 0.
            doc["attn_activation_bytes_per_ctx_token"] = 0.0
        else:
            doc["attn_flops_per_context"] = float(4 * self.n_heads * self.head_dim)
        return doc

    def to_dict(self) -> dict[str, Any]:
        return asdict(self)


TINY = ModelArch(
    name="tiny-mixtral", family="mixtral", vocab=32000, hidden=256, layers=4, n_heads=8, n_kv_heads=2,
    head_dim=32, moe_ffn=512, n_experts=8, top_k=2, rope_theta=1e6, rms_eps=1e-5)

MIXTRAL_8X7B = ModelArch(
    name="mixtral-8x7b", family="mixtral", vocab=32000, hidden=4096, layers=32, n_heads=32, n_kv_heads=8,
    head_dim=128, moe_ffn=14336, n_experts=8, top_k=2, rope_theta=1e6, rms_eps=1e-5)

MIXTRAL_8X22B = ModelArch(
    name="mixtral-8x22b", family="mixtral", vocab=32768, hidden=6144, layers=56, n_heads=48, n_kv_heads=8,
    head_dim=128, moe_ffn=16384, n_experts=8, top_k=2, rope_theta=1e6, rms_eps=1e-5)

DSV2_LITE = ModelArch(
    name="deepseek-v2-lite", family="deepseek_v2", vocab=102400, hidden=2048, layers=27, n_heads=16,
    n_kv_heads=16, head_dim=192, moe_ffn=1408, n_experts=64, top_k=6, rope_theta=10000.0, rms_eps=1e-6,
    n_shared=2, first_k_dense=1, dense_ffn=10944, q_lora_rank=0, kv_lora_rank=512, qk_nope_dim=128,
    qk_rope_dim=64, v_head_dim=128, routed_scaling=1.0, topk_method="greedy")

DSV2_236B = ModelArch(
    name="deepseek-v2-236b", family="deepseek_v2", vocab=102400, hidden=5120, layers=60, n_heads=128,
    n_kv_heads=128, head_dim=192, moe_ffn=1536, n_experts=160, top_k=6, rope_theta=10000.0, rms_eps=1e-6,
    n_shared=2, first_k_dense=1, dense_ffn=12288, q_lora_rank=1536, kv_lora_rank=512, qk_nope_dim=128,
    qk_rope_dim=64, v_head_dim=128, routed_scaling=16.0, topk_method="group_limited_greedy", n_group=8,
    topk_group=3)

TINY_DSV2 = replace(
    DSV2_LITE, name="tiny-deepseek-v2", vocab=4096, hidden=256, layers=3, n_heads=4, n_kv_heads=4,
    moe_ffn=128, n_experts=16, top_k=4, dense_ffn=512, kv_lora_rank=128, qk_nope_dim=32, qk_rope_dim=32,
    v_head_dim=32, head_dim=64, topk_method="group_limited_greedy", n_group=4, topk_group=2,
    routed_scaling=2.0)

ARCHS = {a.name: a for a in (TINY, MIXTRAL_8X7B, MIXTRAL_8X22B, DSV2_LITE, DSV2_236B, TINY_DSV2)}


def get_arch(name: str) -> ModelArch:
    try:
        return ARCHS[name]
    except KeyError:
        raise KeyError(f"unknown architecture {name!r}; available: {', '.join(sorted(ARCHS))}") from None
