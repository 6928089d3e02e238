"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

CPU (torch, bf16) restatement of the MoE decode hot path the B200 engine executes.
The reference (arxiv 2503.09716, /root/reference) ships no numerics for this path
(SPEC.md:20,96): its DAG names the modules (offload_dag.py:62-86) and the paper's engine runs the
HuggingFace model.  The published algorithm restated here is therefore
HF transformers 5.5.0 (third-party, present in this container, not a reference dependency):
  - MixtralTopKRouter.forward       modeling_mixtral.py:109-116
  - MixtralExperts / grouped_mm     modeling_mixtral.py:74-98, integrations/moe.py:350-429
  - MixtralRMSNorm                  modeling_mixtral.py:140-152
  - apply_rotary_pos_emb / rotary   modeling_mixtral.py:210-254
  - eager_attention_forward         modeling_mixtral.py:269-291
  - DeepseekV2Moe.route_tokens_to_experts  modeling_deepseek_v2.py:100-120
with the orders HF leaves unspecified pinned:
  (i)  top-k selection on logits, value descending, lower expert index first on ties;
  (ii) permutation = stable sort of token-major flat entries (t*k+j) by expert;
  (iii) combine = sum_j w[t,j] * y[pos(t,j)] in fp32, j ascending, one bf16 rounding.
Parity is pinned by tests/golden/ fixtures generated from HF itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch
import torch.nn.functional as F

from .rng import uniform_bf16

BF16 = torch.bfloat16

# ---- tensor-id scheme of the counter-based weights (mirrors paper_2503_09716_b200/weights.py) ----
TID_EMBED, TID_FINAL_NORM, TID_LM_HEAD = 1, 2, 3
LAYER_BASE, LAYER_STRIDE = 1000, 100
SLOT = dict(ln1=0, wq=1, wk=2, wv=3, wo=4, ln2=5, router=6, w_gate_up=7, w_down=8)


def tid(layer: int, name: str) -> int:
    return LAYER_BASE + LAYER_STRIDE * layer + SLOT[name]


# ------------------------------------------------------------------------------------------
# routing (pinned orders)
# ------------------------------------------------------------------------------------------
def select_topk(logits: torch.Tensor, k: int, allowed: torch.Tensor | None = None) -> torch.Tensor:
    """Indices of the k best logits per row: value descending, index ascending on ties."""
    lg = logits.float()
    if allowed is not None:
        lg = lg.masked_fill(~allowed, float("-inf"))
    order = torch.sort(-lg, dim=-1, stable=True).indices
    return order[:, :k]


def route(logits: torch.Tensor, k: int, mode: int, scaling: float = 1.0, n_group: int = 1,
          topk_group: int = 1) -> tuple[torch.Tensor, torch.Tensor]:
    """(topk_idx int64 [T,k], topk_w fp32 [T,k]) from router logits.
    mode 0: Mixtral (modeling_mixtral.py:112-115): softmax fp32, top-k, renormalise.
    mode 1: DeepSeek-V2 greedy (modeling_deepseek_v2.py:103-105,118): softmax, top-k, x scaling.
    mode 2: DeepSeek-V2 group_limited_greedy (:106-116): groups ranked by max prob."""
    lg = logits.float()
    probs = torch.softmax(lg, dim=-1)
    allowed = None
    if mode == 2:
        T, E = lg.shape
        gmax = lg.view(T, n_group, E // n_group).max(dim=-1).values
        gsel = select_topk(gmax, topk_group)
        gmask = torch.zeros(T, n_group, dtype=torch.bool)
        gmask.scatter_(1, gsel, True)
        allowed = gmask.unsqueeze(-1).expand(T, n_group, E // n_group).reshape(T, E)
    idx = select_topk(lg, k, allowed)
    w = torch.gather(probs, 1, idx)
    if mode == 0:
        w = w / w.sum(dim=-1, keepdim=True)
    else:
        w = w * scaling
    return idx, w


def permutation(topk_idx: torch.Tensor, E: int):
    """Stable expert-major order of the flat entries.
    Returns (order[T*k]: flat entry at each permuted row, dst_pos[T*k]: permuted row of each
    flat entry, counts[E], offsets[E+1])."""
    flat = topk_idx.reshape(-1)
    order = torch.sort(flat, stable=True).indices
    dst = torch.empty_like(order)
    dst[order] = torch.arange(order.numel())
    counts = torch.bincount(flat, minlength=E)
    offsets = torch.zeros(E + 1, dtype=torch.int64)
    offsets[1:] = torch.cumsum(counts, 0)
    return order, dst, counts, offsets


def expert_ffn(x: torch.Tensor, w_gate_up: torch.Tensor, w_down: torch.Tensor) -> torch.Tensor:
    """MixtralExperts per-expert math (modeling_mixtral.py:90-94) in bf16."""
    gate, up = F.linear(x, w_gate_up).chunk(2, dim=-1)
    h = F.silu(gate) * up
    return F.linear(h, w_down)


def moe_block(x: torch.Tensor, w_router: torch.Tensor, w_gate_up: torch.Tensor, w_down: torch.Tensor,
              k: int, mode: int = 0, scaling: float = 1.0, n_group: int = 1, topk_group: int = 1,
              fp32_router: bool = False, trace: dict | None = None) -> torch.Tensor:
    """Routed-expert output (before residual) for x[T,d] bf16."""
    T, d = x.shape
    E = w_router.shape[0]
    if fp32_router:
        logits = F.linear(x.float(), w_router.float())
    else:
        logits = F.linear(x, w_router)  # bf16 GEMM (modeling_mixtral.py:111)
    idx, w = route(logits, k, mode, scaling, n_group, topk_group)
    order, dst, counts, offsets = permutation(idx, E)
    tok_of_row = order // k
    xp = x[tok_of_row]
    yp = torch.empty(T * k, d, dtype=BF16)
    for e in range(E):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if b > a:
            yp[a:b] = expert_ffn(xp[a:b], w_gate_up[e], w_down[e])
    acc = torch.zeros(T, d, dtype=torch.float32)
    for j in range(k):
        acc += yp[dst.view(T, k)[:, j]].float() * w[:, j:j + 1]
    out = acc.to(BF16)
    if trace is not None:
        trace.update(logits=logits, topk_idx=idx, topk_w=w, order=order, dst_pos=dst, counts=counts,
                     offsets=offsets, x_perm=xp, y_perm=yp, moe_out=out)
    return out


# ------------------------------------------------------------------------------------------
# dense pieces
# ------------------------------------------------------------------------------------------
def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    h = x.float()
    var = h.pow(2).mean(-1, keepdim=True)
    h = h * torch.rsqrt(var + eps)
    return w * h.to(x.dtype)


def rope_cos_sin(theta: float, hd: int, positions: torch.Tensor) -> tuple[torch.Tensor, torch.Tensor]:
    inv_freq = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    freqs = positions.float()[:, None] * inv_freq[None, :]
    emb = torch.cat((freqs, freqs), dim=-1)
    return emb.cos().to(BF16), emb.sin().to(BF16)


def rotate_half(x):
    x1 = x[..., : x.shape[-1] // 2]
    x2 = x[..., x.shape[-1] // 2:]
    return torch.cat((-x2, x1), dim=-1)


def apply_rope(x: torch.Tensor, cos: torch.Tensor, sin: torch.Tensor) -> torch.Tensor:
    """x [T, H, hd]; cos/sin [T, hd] (bf16)."""
    return (x * cos[:, None, :]) + (rotate_half(x) * sin[:, None, :])


def gqa_decode_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, impl: str = "sdpa") -> torch.Tensor:
    """Decode attention for one query token per sequence; q [B, Hq, hd]; k, v [B, Hkv, ctx, hd]
    -> [B, Hq*hd].  KV head of query head i is i // G (repeat_kv, modeling_mixtral.py:257-266).
    impl="sdpa" (HF's default attn_implementation): scores, softmax and P.V in fp32, one bf16
    rounding of the output.  impl="eager" (modeling_mixtral.py:269-291): bf16 scores and bf16 P."""
    B, Hq, hd = q.shape
    if B > 128:  # bounded temporaries at bench batch sizes (sequences are independent)
        return torch.cat([gqa_decode_attention(q[b:b + 128], k[b:b + 128], v[b:b + 128], impl)
                          for b in range(0, B, 128)])
    G = Hq // k.shape[1]
    kk = k.repeat_interleave(G, dim=1)
    vv = v.repeat_interleave(G, dim=1)
    if impl == "eager":
        scores = torch.matmul(q[:, :, None, :], kk.transpose(2, 3)) * (hd ** -0.5)
        p = torch.softmax(scores, dim=-1, dtype=torch.float32).to(q.dtype)
        o = torch.matmul(p, vv)  # [B, Hq, 1, hd]
        return o.reshape(B, Hq * hd)
    scores = torch.matmul(q[:, :, None, :].float(), kk.float().transpose(2, 3)) * (hd ** -0.5)
    p = torch.softmax(scores, dim=-1)
    o = torch.matmul(p, vv.float())
    return o.reshape(B, Hq * hd).to(q.dtype)


# ------------------------------------------------------------------------------------------
# Mixtral-family model (decode-only, equal-length sequences)
# ------------------------------------------------------------------------------------------
@dataclass
class MixtralWeights:
    embed: torch.Tensor
    final_norm: torch.Tensor
    lm_head: torch.Tensor
    layers: list


def make_mixtral_weights(arch, seed: int = 0) -> MixtralWeights:
    """Counter-based random init identical to the device generator (oracle/rng.py)."""
    d, hd = arch.hidden, arch.head_dim
    std = arch.init_std
    U = lambda shape, t: uniform_bf16(shape, seed, t, std)  # noqa: E731
    layers = []
    for l in range(arch.layers):
        layers.append(dict(
            ln1=torch.ones(d, dtype=BF16),
            wq=U((arch.n_heads * hd, d), tid(l, "wq")),
            wk=U((arch.n_kv_heads * hd, d), tid(l, "wk")),
            wv=U((arch.n_kv_heads * hd, d), tid(l, "wv")),
            wo=U((d, arch.n_heads * hd), tid(l, "wo")),
            ln2=torch.ones(d, dtype=BF16),
            router=U((arch.n_experts, d), tid(l, "router")),
            w_gate_up=U((arch.n_experts, 2 * arch.moe_ffn, d), tid(l, "w_gate_up")),
            w_down=U((arch.n_experts, d, arch.moe_ffn), tid(l, "w_down")),
        ))
    return MixtralWeights(
        embed=U((arch.vocab, d), TID_EMBED),
        final_norm=torch.ones(d, dtype=BF16),
        lm_head=U((arch.vocab, d), TID_LM_HEAD),
        layers=layers,
    )


class MixtralOracle:
    """Token-by-token greedy decoding of B equal-length sequences on the CPU."""

    def __init__(self, arch, weights: MixtralWeights):
        self.a = arch
        self.w = weights
        self.k_cache = [None] * arch.layers  # [B, Hkv, ctx, hd]
        self.v_cache = [None] * arch.layers

    def set_kv(self, layer: int, k: torch.Tensor, v: torch.Tensor) -> None:
        self.k_cache[layer], self.v_cache[layer] = k, v

    def layer_forward(self, l: int, x: torch.Tensor, pos: int, trace: dict | None = None) -> torch.Tensor:
        a, W = self.a, self.w.layers[l]
        B = x.shape[0]
        hd = a.head_dim
        h = rmsnorm(x, W["ln1"], a.rms_eps)
        q = F.linear(h, W["wq"]).view(B, a.n_heads, hd)
        kk = F.linear(h, W["wk"]).view(B, a.n_kv_heads, hd)
        vv = F.linear(h, W["wv"]).view(B, a.n_kv_heads, hd)
        cos, sin = rope_cos_sin(a.rope_theta, hd, torch.full((B,), pos))
        q = apply_rope(q, cos, sin)
        kk = apply_rope(kk, cos, sin)
        if self.k_cache[l] is None:
            self.k_cache[l] = kk[:, :, None, :]
            self.v_cache[l] = vv[:, :, None, :]
        else:
            self.k_cache[l] = torch.cat([self.k_cache[l], kk[:, :, None, :]], dim=2)
            self.v_cache[l] = torch.cat([self.v_cache[l], vv[:, :, None, :]], dim=2)
        attn = gqa_decode_attention(q, self.k_cache[l], self.v_cache[l])
        x = x + F.linear(attn, W["wo"])
        h2 = rmsnorm(x, W["ln2"], a.rms_eps)
        moe = moe_block(h2, W["router"], W["w_gate_up"], W["w_down"], a.top_k, 0, trace=trace)
        if trace is not None:
            trace.update(attn=attn, h2=h2, q=q)
        return x + moe

    def step(self, tokens: torch.Tensor, pos: int, traces: list | None = None) -> torch.Tensor:
        """One decode step; tokens [B] int64 at position `pos` -> logits [B, V] bf16."""
        x = self.w.embed[tokens]
        for l in range(self.a.layers):
            tr = {} if traces is not None else None
            x = self.layer_forward(l, x, pos, tr)
            if traces is not None:
                tr["x_out"] = x
                traces.append(tr)
        h = rmsnorm(x, self.w.final_norm, self.a.rms_eps)
        return F.linear(h, self.w.lm_head)

    def generate(self, input_ids: torch.Tensor, max_new_tokens: int) -> tuple[torch.Tensor, list]:
        """Greedy; the prompt is consumed token by token.  Returns (ids [B, P+N], step logits)."""
        B, P = input_ids.shape
        ids = input_ids.clone()
        logits_all = []
        cur = None
        for p in range(P):
            cur = self.step(ids[:, p], p)
        for n in range(max_new_tokens):
            nxt = torch.argmax(cur.float(), dim=-1)
            logits_all.append(cur)
            ids = torch.cat([ids, nxt[:, None]], dim=1)
            if n + 1 < max_new_tokens:
                cur = self.step(nxt, P + n)
        return ids, logits_all


def rel_err(a: torch.Tensor, b: torch.Tensor) -> float:
    """max|a-b| / max|b| (the per-layer tolerance metric of BASELINE.json north_star)."""
    a, b = a.float(), b.float()
    den = b.abs().max().item()
    return (a - b).abs().max().item() / (den if den > 0 else 1.0)


def cosine(a: torch.Tensor, b: torch.Tensor) -> float:
    a, b = a.float().reshape(-1), b.float().reshape(-1)
    return float(torch.dot(a, b) / (a.norm() * b.norm() + 1e-30))


def softmax_margin(logits: torch.Tensor) -> torch.Tensor:
    top2 = torch.topk(logits.float(), 2, dim=-1).values
    return top2[:, 0] - top2[:, 1]


__all__ = [n for n in dir() if not n.startswith("_")] + ["math"]


# ------------------------------------------------------------------------------------------
# DeepSeek-V2 family (MLA attention, shared experts, dense first layers)
# HF transformers 5.5.0 modeling_deepseek_v2.py: DeepseekV2Attention.forward :337-396,
# apply_rotary_emb :305-318, DeepseekV2Moe :85-131, DeepseekV2MLP :134-146, decoder layer :399-430
# ------------------------------------------------------------------------------------------
DS_SLOT = dict(ln1=0, ln2=5, router=6, w_gate_up=7, w_down=8, q_proj=10, q_a_norm=11, q_b=12, kv_a=13,
               kv_a_norm=14, kv_b=15, wo=16, sh_gate_up=17, sh_down=18, dense_gate_up=19, dense_down=20)


def ds_tid(layer: int, name: str) -> int:
    return LAYER_BASE + LAYER_STRIDE * layer + DS_SLOT[name]


def make_dsv2_weights(arch, seed: int = 0) -> MixtralWeights:
    a = arch
    d, H = a.hidden, a.n_heads
    qk = a.qk_nope_dim + a.qk_rope_dim
    std = a.init_std
    U = lambda shape, t: uniform_bf16(shape, seed, t, std)  # noqa: E731
    ones = lambda n: torch.ones(n, dtype=BF16)  # noqa: E731
    layers = []
    for l in range(a.layers):
        L = dict(ln1=ones(d), ln2=ones(d),
                 kv_a=U((a.kv_lora_rank + a.qk_rope_dim, d), ds_tid(l, "kv_a")), kv_a_norm=ones(a.kv_lora_rank),
                 kv_b=U((H * (a.qk_nope_dim + a.v_head_dim), a.kv_lora_rank), ds_tid(l, "kv_b")),
                 wo=U((d, H * a.v_head_dim), ds_tid(l, "wo")))
        if a.q_lora_rank:
            L.update(q_a=U((a.q_lora_rank, d), ds_tid(l, "q_proj")), q_a_norm=ones(a.q_lora_rank),
                     q_b=U((H * qk, a.q_lora_rank), ds_tid(l, "q_b")))
        else:
            L.update(q_proj=U((H * qk, d), ds_tid(l, "q_proj")))
        if l < a.first_k_dense:
            L.update(dense_gate_up=U((2 * a.dense_ffn, d), ds_tid(l, "dense_gate_up")),
                     dense_down=U((d, a.dense_ffn), ds_tid(l, "dense_down")))
        else:
            fs = a.moe_ffn * a.n_shared
            L.update(router=U((a.n_experts, d), ds_tid(l, "router")),
                     w_gate_up=U((a.n_experts, 2 * a.moe_ffn, d), ds_tid(l, "w_gate_up")),
                     w_down=U((a.n_experts, d, a.moe_ffn), ds_tid(l, "w_down")),
                     sh_gate_up=U((2 * fs, d), ds_tid(l, "sh_gate_up")), sh_down=U((d, fs), ds_tid(l, "sh_down")))
        layers.append(L)
    return MixtralWeights(embed=U((a.vocab, d), TID_EMBED), final_norm=ones(d), lm_head=U((a.vocab, d), TID_LM_HEAD),
                          layers=layers)


def rope_interleaved(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    """apply_rotary_emb (modeling_deepseek_v2.py:305-318): complex rotation of (2i, 2i+1) pairs in
    fp32, one cast back.  x [T, H, r], pos [T]."""
    r = x.shape[-1]
    inv_freq = 1.0 / (theta ** (torch.arange(0, r, 2, dtype=torch.int64).float() / r))
    freqs = pos.float()[:, None] * inv_freq[None, :]
    cis = torch.polar(torch.ones_like(freqs), freqs)  # [T, r/2]
    xc = torch.view_as_complex(x.float().reshape(*x.shape[:-1], -1, 2))
    return torch.view_as_real(xc * cis[:, None, :]).flatten(-2).type_as(x)


def mla_absorbed_attention(q_lat: torch.Tensor, q_pe: torch.Tensor, c_cache: torch.Tensor, pe_cache: torch.Tensor,
                           scale: float) -> torch.Tensor:
    """Absorbed MLA decode attention in fp32 (what mgb_decode_attn_mla computes):
    q_lat [B,H,R], q_pe [B,H,r]; c_cache [B,ctx,R], pe_cache [B,ctx,r] -> o_lat [B,H,R] (bf16)."""
    s = (torch.einsum("bhr,btr->bht", q_lat.float(), c_cache.float())
         + torch.einsum("bhr,btr->bht", q_pe.float(), pe_cache.float())) * scale
    p = torch.softmax(s, dim=-1)
    return torch.einsum("bht,btr->bhr", p, c_cache.float()).to(q_lat.dtype)


class DeepseekV2Oracle:
    """Token-by-token greedy decoding (HF DeepseekV2 semantics, non-absorbed attention with
    per-head K/V caches, sdpa-style fp32 attention)."""

    def __init__(self, arch, weights: MixtralWeights):
        self.a, self.w = arch, weights
        self.kc = [None] * arch.layers
        self.vc = [None] * arch.layers
        # latent caches (c [B, ctx, R] normed, k_pe [B, ctx, r] rotated): when set for a layer, that
        # layer attends in the latent form (`_latent_attention`) instead of per-head K/V caches
        self.lat = [None] * arch.layers

    def set_latent(self, layer: int, c: torch.Tensor, k_pe: torch.Tensor) -> None:
        self.lat[layer] = (c, k_pe)

    def _latent_attention(self, l: int, query_nope, q_pe, c, k_pe, B: int) -> torch.Tensor:
        """HF DeepseekV2Attention (modeling_deepseek_v2.py:337-396) over a latent cache, evaluated
        in fp32 by associativity instead of materialising per-head K/V for the whole context:
        q.k_h = (q_nope W_UK_h) . c + q_pe . k_pe and o_h = (P c) W_UV_h^T, with
        kv_b_proj = [W_UK_h ; W_UV_h] per head (:356-370).  Exact arithmetic equals HF's; HF rounds
        k_nope / v to bf16 first, which the bf16 tolerance covers.  One bf16 rounding of o."""
        a, W = self.a, self.w.layers[l]
        H, nope, rope, vd, R = a.n_heads, a.qk_nope_dim, a.qk_rope_dim, a.v_head_dim, a.kv_lora_rank
        c0, pe0 = self.lat[l]
        self.lat[l] = (torch.cat([c0, c[:, None]], 1), torch.cat([pe0, k_pe.view(B, 1, rope)], 1))
        cc, pp = self.lat[l]
        kvb = W["kv_b"].float().view(H, nope + vd, R)
        w_uk, w_uv = kvb[:, :nope], kvb[:, nope:]                     # [H, nope, R], [H, vd, R]
        scale = (nope + rope) ** -0.5
        out = torch.empty(B, H, vd)
        for b0 in range(0, B, 256):                                   # bounded fp32 temporaries
            b1 = min(B, b0 + 256)
            q_lat = torch.einsum("bhn,hnr->bhr", query_nope[b0:b1].float(), w_uk)
            s = (torch.einsum("bhr,btr->bht", q_lat, cc[b0:b1].float())
                 + torch.einsum("bhr,btr->bht", q_pe[b0:b1].float(), pp[b0:b1].float())) * scale
            o_lat = torch.einsum("bht,btr->bhr", torch.softmax(s, dim=-1), cc[b0:b1].float())
            out[b0:b1] = torch.einsum("bhr,hvr->bhv", o_lat, w_uv)
        return out.reshape(B, H * vd).to(BF16)

    def attention(self, l: int, h: torch.Tensor, pos: int, trace: dict | None = None) -> torch.Tensor:
        a, W = self.a, self.w.layers[l]
        B, H = h.shape[0], a.n_heads
        nope, rope, vd = a.qk_nope_dim, a.qk_rope_dim, a.v_head_dim
        if a.q_lora_rank:
            q = F.linear(rmsnorm(F.linear(h, W["q_a"]), W["q_a_norm"], a.rms_eps), W["q_b"])
        else:
            q = F.linear(h, W["q_proj"])
        q = q.view(B, H, nope + rope)
        q_nope, q_pe = q[..., :nope], q[..., nope:]
        ckv = F.linear(h, W["kv_a"])
        c, k_pe = ckv[:, :a.kv_lora_rank], ckv[:, a.kv_lora_rank:]
        c = rmsnorm(c, W["kv_a_norm"], a.rms_eps)
        posv = torch.full((B,), pos)
        if self.lat[l] is not None:
            q_pe = rope_interleaved(q_pe, posv, a.rope_theta)
            k_pe = rope_interleaved(k_pe.view(B, 1, rope), posv, a.rope_theta).view(B, rope)
            o = self._latent_attention(l, q_nope, q_pe, c, k_pe, B)
            if trace is not None:
                trace.update(c=c, k_pe=k_pe, q_nope=q_nope, q_pe=q_pe, attn=o)
            return F.linear(o, W["wo"])
        kvb = F.linear(c, W["kv_b"]).view(B, H, nope + vd)
        k_nope, v = kvb[..., :nope], kvb[..., nope:]
        q_pe = rope_interleaved(q_pe, posv, a.rope_theta)
        k_pe = rope_interleaved(k_pe.view(B, 1, rope), posv, a.rope_theta)
        key = torch.cat([k_nope, k_pe.expand(B, H, rope)], dim=-1)
        query = torch.cat([q_nope, q_pe], dim=-1)
        if self.kc[l] is None:
            self.kc[l], self.vc[l] = key[:, :, None], v[:, :, None]
        else:
            self.kc[l] = torch.cat([self.kc[l], key[:, :, None]], 2)
            self.vc[l] = torch.cat([self.vc[l], v[:, :, None]], 2)
        scale = (nope + rope) ** -0.5
        s = torch.matmul(query[:, :, None, :].float(), self.kc[l].float().transpose(2, 3)) * scale
        p = torch.softmax(s, dim=-1)
        o = torch.matmul(p, self.vc[l].float()).reshape(B, H * vd).to(h.dtype)
        if trace is not None:
            trace.update(c=c, k_pe=k_pe.view(B, rope), q_nope=q_nope, q_pe=q_pe, attn=o)
        return F.linear(o, W["wo"])

    def layer_forward(self, l: int, x: torch.Tensor, pos: int, trace: dict | None = None) -> torch.Tensor:
        a, W = self.a, self.w.layers[l]
        h = rmsnorm(x, W["ln1"], a.rms_eps)
        x = x + self.attention(l, h, pos, trace)
        h2 = rmsnorm(x, W["ln2"], a.rms_eps)
        if l < a.first_k_dense:
            y = expert_ffn(h2, W["dense_gate_up"], W["dense_down"])
        else:
            routed = moe_block(h2, W["router"], W["w_gate_up"], W["w_down"], a.top_k, a.router_mode, a.routed_scaling,
                               a.n_group, a.topk_group, fp32_router=True, trace=trace)
            y = routed + expert_ffn(h2, W["sh_gate_up"], W["sh_down"])
        if trace is not None:
            trace.update(h2=h2)
        return x + y

    def step(self, tokens: torch.Tensor, pos: int, traces: list | None = None) -> torch.Tensor:
        x = self.w.embed[tokens]
        for l in range(self.a.layers):
            tr = {} if traces is not None else None
            x = self.layer_forward(l, x, pos, tr)
            if traces is not None:
                tr["x_out"] = x
                traces.append(tr)
        return F.linear(rmsnorm(x, self.w.final_norm, self.a.rms_eps), self.w.lm_head)

    def generate(self, input_ids: torch.Tensor, max_new_tokens: int):
        B, P = input_ids.shape
        ids = input_ids.clone()
        cur = None
        for p in range(P):
            cur = self.step(ids[:, p], p)
        for n in range(max_new_tokens):
            nxt = torch.argmax(cur.float(), dim=-1)
            ids = torch.cat([ids, nxt[:, None]], dim=1)
            if n + 1 < max_new_tokens:
                cur = self.step(nxt, P + n)
        return ids
