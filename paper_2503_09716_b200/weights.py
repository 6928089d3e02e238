"""Device-resident random-init weights, generated in HBM by the counter-based kernel
(mgb_fill_uniform_bf16) so 93-471 GB models need no host files and are bit-identical to the
CPU oracle's copy (oracle/rng.py) at small sizes.

Tensor-id scheme (must match oracle/moe_ref.py): globals 1 embed, 2 final norm, 3 lm_head;
layer l uses 1000 + 100*l + slot.
"""

from __future__ import annotations

import torch

from . import _native as nat
from .configs import ModelArch

TID_EMBED, TID_FINAL_NORM, TID_LM_HEAD = 1, 2, 3
LAYER_BASE, LAYER_STRIDE = 1000, 100
SLOT = dict(ln1=0, wq=1, wk=2, wv=3, wo=4, ln2=5, router=6, w_gate_up=7, w_down=8)


def tid(layer: int, name: str) -> int:
    return LAYER_BASE + LAYER_STRIDE * layer + SLOT[name]


def fill_uniform_(t: torch.Tensor, seed: int, tensor_id: int, std: float, first: int = 0) -> torch.Tensor:
    """t <- elements [first, first + t.numel()) of tensor `tensor_id`'s counter-based stream."""
    assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous()
    if first:
        nat.call("mgb_fill_uniform_bf16_range", t.data_ptr(), t.numel(), first, seed, tensor_id, std,
                 torch.cuda.current_stream().cuda_stream)
    else:
        nat.call("mgb_fill_uniform_bf16", t.data_ptr(), t.numel(), seed, tensor_id, std, 0.0, 0,
                 torch.cuda.current_stream().cuda_stream)
    return t


def routed_experts_(a: ModelArch, seed: int, tid_gate_up: int, tid_down: int, device: str,
                    experts: tuple[int, int] | None) -> tuple[torch.Tensor, torch.Tensor]:
    """Routed expert weights [n, 2f, d] / [n, d, f] of experts [lo, lo + n) (all when experts is None),
    generated in place: an expert-parallel rank never holds the other ranks' experts."""
    lo, n = experts if experts is not None else (0, a.n_experts)
    f, d = a.moe_ffn, a.hidden
    bf = dict(dtype=torch.bfloat16, device=device)
    gu = fill_uniform_(torch.empty(n, 2 * f, d, **bf), seed, tid_gate_up, a.init_std, first=lo * 2 * f * d)
    dn = fill_uniform_(torch.empty(n, d, f, **bf), seed, tid_down, a.init_std, first=lo * d * f)
    return gu, dn


def _shard_source(L: dict, experts: tuple[int, int] | None) -> dict:
    """A checkpoint layer restricted to the rank's routed experts (before it moves to the device)."""
    if experts is not None and L.get("w_gate_up") is not None:
        lo, n = experts
        L = dict(L, w_gate_up=L["w_gate_up"][lo:lo + n], w_down=L["w_down"][lo:lo + n])
    return L


def fill_const_(t: torch.Tensor, value: float) -> torch.Tensor:
    assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous()
    nat.call("mgb_fill_uniform_bf16", t.data_ptr(), t.numel(), 0, 0, 0.0, value, 1,
             torch.cuda.current_stream().cuda_stream)
    return t


def mixtral_layer(a: ModelArch, l: int, seed: int, device: str = "cuda", source=None,
                  experts: tuple[int, int] | None = None) -> dict:
    """Layer l of a Mixtral-family model in the engine's layout.  q/k/v projections are stored
    fused as one [Hq*hd + 2*Hkv*hd, d] matrix (rows = wq | wk | wv), each part generated with its
    own tensor id so it equals the oracle's separate wq/wk/wv.  `source` (checkpoint.Checkpoint)
    loads the layer from a safetensors checkpoint instead of generating it.  experts=(lo, n): only
    routed experts [lo, lo + n) (an expert-parallel rank's shard)."""
    if source is not None:
        return {k: v.to(device) for k, v in _shard_source(source.layer(l), experts).items()}
    d, hd = a.hidden, a.head_dim
    qd, kvd = a.n_heads * hd, a.n_kv_heads * hd
    std = a.init_std
    bf = dict(dtype=torch.bfloat16, device=device)
    wqkv = torch.empty(qd + 2 * kvd, d, **bf)
    fill_uniform_(wqkv[:qd], seed, tid(l, "wq"), std)
    fill_uniform_(wqkv[qd:qd + kvd], seed, tid(l, "wk"), std)
    fill_uniform_(wqkv[qd + kvd:], seed, tid(l, "wv"), std)
    w_gate_up, w_down = routed_experts_(a, seed, tid(l, "w_gate_up"), tid(l, "w_down"), device, experts)
    return dict(
        ln1=fill_const_(torch.empty(d, **bf), 1.0),
        wqkv=wqkv,
        wo=fill_uniform_(torch.empty(d, qd, **bf), seed, tid(l, "wo"), std),
        ln2=fill_const_(torch.empty(d, **bf), 1.0),
        router=fill_uniform_(torch.empty(a.n_experts, d, **bf), seed, tid(l, "router"), std),
        w_gate_up=w_gate_up,
        w_down=w_down,
    )


class _DeviceWeights:
    """All weights HBM-resident, generated layer by layer by the family's layer builder."""

    def __init__(self, arch: ModelArch, seed: int = 0, device: str = "cuda", source=None,
                 experts: tuple[int, int] | None = None):
        a = arch
        self.arch = a
        self.experts = experts  # (lo, n): this rank's routed-expert shard; None = all experts
        self.embed, self.final_norm, self.lm_head = global_tensors(a, seed, device, source)
        build = deepseek_layer if a.is_mla else mixtral_layer
        self.layers = [build(a, l, seed, device, source, experts) for l in range(a.layers)]

    def nbytes(self) -> int:
        n = self.embed.nbytes + self.final_norm.nbytes + self.lm_head.nbytes
        for L in self.layers:
            n += sum(t.nbytes for k, t in L.items() if k not in DERIVED)
        return n


def global_tensors(a: ModelArch, seed: int, device: str, source=None):
    """(embed, final norm, lm_head): generated, or loaded from a checkpoint `source`."""
    if source is not None:
        return source.embed().to(device), source.final_norm().to(device), source.lm_head().to(device)
    bf = dict(dtype=torch.bfloat16, device=device)
    return (fill_uniform_(torch.empty(a.vocab, a.hidden, **bf), seed, TID_EMBED, a.init_std),
            fill_const_(torch.empty(a.hidden, **bf), 1.0),
            fill_uniform_(torch.empty(a.vocab, a.hidden, **bf), seed, TID_LM_HEAD, a.init_std))


class MixtralDeviceWeights(_DeviceWeights):
    pass


class DeepseekDeviceWeights(_DeviceWeights):
    pass


DS_SLOT = dict(ln1=0, ln2=5, router=6, w_gate_up=7, w_down=8, q_proj=10, q_a_norm=11, q_b=12, kv_a=13,
               kv_a_norm=14, kv_b=15, wo=16, sh_gate_up=17, sh_down=18, dense_gate_up=19, dense_down=20)


def ds_tid(layer: int, name: str) -> int:
    return LAYER_BASE + LAYER_STRIDE * layer + DS_SLOT[name]


def deepseek_layer(a: ModelArch, l: int, seed: int, device: str = "cuda", source=None,
                   experts: tuple[int, int] | None = None) -> dict:
    """Layer l of a DeepSeek-V2-family model in HF layouts (q_proj or q_a/q_b, kv_a_proj_with_mqa,
    kv_b_proj, o_proj; routed experts [E,2f,d]/[E,d,f]; shared experts and the dense first layers
    as fused gate|up [2f,d] + down [d,f]).  Tensor ids mirror oracle/moe_ref.py DS_SLOT.
    experts=(lo, n): only routed experts [lo, lo + n) (an expert-parallel rank's shard)."""
    if source is not None:
        return derive_views(a, {k: v.to(device) for k, v in _shard_source(source.layer(l), experts).items()})
    d, H = a.hidden, a.n_heads
    qk = a.qk_nope_dim + a.qk_rope_dim
    std = a.init_std
    bf = dict(dtype=torch.bfloat16, device=device)
    U = lambda shape, name: fill_uniform_(torch.empty(*shape, **bf), seed, ds_tid(l, name), std)  # noqa: E731
    ones = lambda n: fill_const_(torch.empty(n, **bf), 1.0)  # noqa: E731
    L = dict(ln1=ones(d), ln2=ones(d), kv_a=U((a.kv_lora_rank + a.qk_rope_dim, d), "kv_a"),
             kv_a_norm=ones(a.kv_lora_rank), kv_b=U((H * (a.qk_nope_dim + a.v_head_dim), a.kv_lora_rank), "kv_b"),
             wo=U((d, H * a.v_head_dim), "wo"))
    if a.q_lora_rank:
        L.update(q_a=U((a.q_lora_rank, d), "q_proj"), q_a_norm=ones(a.q_lora_rank), q_b=U((H * qk, a.q_lora_rank), "q_b"))
    else:
        L["q_proj"] = U((H * qk, d), "q_proj")
    if l < a.first_k_dense:
        L.update(dense_gate_up=U((1, 2 * a.dense_ffn, d), "dense_gate_up"),
                 dense_down=U((1, d, a.dense_ffn), "dense_down"))
    else:
        fs = a.moe_ffn * a.n_shared
        w_gate_up, w_down = routed_experts_(a, seed, ds_tid(l, "w_gate_up"), ds_tid(l, "w_down"), device, experts)
        L.update(router=U((a.n_experts, d), "router"), w_gate_up=w_gate_up, w_down=w_down,
                 sh_gate_up=U((1, 2 * fs, d), "sh_gate_up"), sh_down=U((1, d, fs), "sh_down"))
    derive_views(a, L)
    return L


DERIVED = ("w_uk", "w_uv_t")


def derive_views(a: ModelArch, L: dict) -> dict:
    """Absorption views of kv_b_proj: rows [h*(nope+v), h*(nope+v)+nope) = W_UK_h, rest = W_UV_h."""
    if a.is_mla:
        kvb = L["kv_b"].view(a.n_heads, a.qk_nope_dim + a.v_head_dim, a.kv_lora_rank)
        L["w_uk"] = kvb[:, :a.qk_nope_dim, :]                     # [H, nope, R]
        L["w_uv_t"] = kvb[:, a.qk_nope_dim:, :].transpose(1, 2)   # [H, R, v]
    return L


def dense_keys(a: ModelArch) -> list[str]:
    """The per-layer 'dense' modules of the reference's memory model (attention weights + shared
    experts, model_catalog.py:55-88 dense_bytes_per_layer): streamed through the single dense
    buffer when the layer is not cached."""
    if not a.is_mla:
        return ["wqkv", "wo"]
    q = ["q_a", "q_b"] if a.q_lora_rank else ["q_proj"]
    return q + ["kv_a", "kv_b", "wo", "sh_gate_up", "sh_down"]
