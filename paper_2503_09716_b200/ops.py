"""Torch-tensor front end of the C-ABI (include/mgb.h).  Every op launches on the current CUDA
stream (so it is CUDA-graph capturable), writes into caller-provided outputs where given, and
raises if the native library is missing or returns an error.  No CPU fallback exists.
"""

from __future__ import annotations

import torch

from . import _native as nat

BF16 = torch.bfloat16


def _s() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_cuda, "device tensor expected"
    return t.data_ptr()


class RouterWorkspace:
    """Router/permutation scratch for up to T tokens and E experts with top-k."""

    def __init__(self, T: int, E: int, k: int, device="cuda"):
        nblk = nat.value("mgb_router_num_blocks", T)
        i32 = dict(dtype=torch.int32, device=device)
        self.T, self.E, self.k = T, E, k
        self.topk_idx = torch.zeros(T, k, **i32)
        self.topk_w = torch.zeros(T, k, dtype=torch.float32, device=device)
        self.local_rank = torch.zeros(T * k, **i32)
        self.block_hist = torch.zeros(nblk, E, **i32)
        self.counts = torch.zeros(E, **i32)
        self.offsets = torch.zeros(E + 1, **i32)
        self.ticket = torch.zeros(1, **i32)
        self.src_token = torch.zeros(T * k, **i32)
        self.dst_pos = torch.zeros(T * k, **i32)
        self.sync = torch.zeros(2, **i32)  # grid barrier of mgb_moe_route
        assert nblk >= nat.value("mgb_moe_route_chunks", T)  # block_hist doubles as its chunk_hist


def router_topk(x: torch.Tensor | None, w_gate: torch.Tensor | None, ws: RouterWorkspace, k: int, mode: int,
                scaling: float = 1.0, n_group: int = 1, topk_group: int = 1,
                logits_in: torch.Tensor | None = None, logits_out: torch.Tensor | None = None,
                T: int | None = None, E: int | None = None) -> None:
    if logits_in is not None:
        T, E = logits_in.shape
        d = 0
    else:
        T, d = x.shape
        E = w_gate.shape[0]
    nat.call("mgb_router_topk", _p(x), _p(w_gate), _p(logits_in), T, d, E, k, mode, scaling, n_group, topk_group,
             _p(logits_out), _p(ws.topk_idx), _p(ws.topk_w), _p(ws.local_rank), _p(ws.block_hist), _p(ws.counts),
             _p(ws.offsets), _p(ws.ticket), _s())


def moe_route_supported(T: int, d: int, E: int) -> bool:
    return bool(nat.value("mgb_moe_route_supported", T, d, E))


def moe_route_single_pass(T: int, d: int, E: int) -> bool:
    """mgb_moe_route covers T tokens with one chunk per CTA (its h_out may be None)."""
    return nat.value("mgb_moe_route_supported", T, d, E) == 2


def moe_route(x: torch.Tensor, delta: torch.Tensor | None, ln_w: torch.Tensor, eps: float, h_out: torch.Tensor | None,
              w_router: torch.Tensor, ws: RouterWorkspace, x_perm: torch.Tensor, mode: int, scaling: float = 1.0,
              n_group: int = 1, topk_group: int = 1, x_out: torch.Tensor | None = None,
              logits_out: torch.Tensor | None = None) -> None:
    """Fused decode routing front end (route.cu): x_out = x + delta, h_out = RMSNorm(x_out) * ln_w,
    top-k routing of h_out, and the stable expert-major permutation of h_out into x_perm.  h_out may be
    None when moe_route_single_pass(T, d, E) (the normalised rows then exist only in x_perm)."""
    T, d = x.shape
    E = w_router.shape[0]
    nat.call("mgb_moe_route", _p(x), _p(delta), _p(ln_w), eps, T, d, _p(x_out), _p(h_out), _p(w_router), E, ws.k,
             mode, scaling, n_group, topk_group, _p(logits_out), _p(ws.topk_idx), _p(ws.topk_w), _p(ws.local_rank),
             _p(ws.block_hist), _p(ws.counts), _p(ws.offsets), _p(x_perm), _p(ws.src_token), _p(ws.dst_pos),
             _p(ws.sync), _s())


def permute(x: torch.Tensor, ws: RouterWorkspace, x_perm: torch.Tensor, T: int | None = None) -> None:
    T = x.shape[0] if T is None else T
    nat.call("mgb_permute", _p(x), _p(ws.topk_idx), _p(ws.local_rank), _p(ws.block_hist), _p(ws.offsets), T,
             x.shape[1], ws.k, ws.E, _p(x_perm), _p(ws.src_token), _p(ws.dst_pos), _s())


class CapacityError(RuntimeError):
    """A grouped launch's row segments exceed the buffer they land in (MGB_ECAPACITY); `counts`
    are the per-expert rows (pre-flight) or {needed, rows_cap, site} (recorded on the device)."""

    def __init__(self, msg: str, counts=None, needed: int = 0, rows_cap: int = 0, site: int = 0):
        super().__init__(msg)
        self.counts, self.needed, self.rows_cap, self.site = counts, needed, rows_cap, site


def check_capacity(offsets: torch.Tensor, rows_cap: int) -> list[int]:
    """Host pre-flight of a grouped launch (synchronises the current stream): per-expert row counts,
    or CapacityError when offsets[E] > rows_cap -- the scheduler then re-splits by b_e."""
    import ctypes

    E = offsets.numel() - 1
    counts = (ctypes.c_int * E)()
    rc = nat.raw("mgb_moe_check_capacity", _p(offsets), E, rows_cap, counts, _s())
    out = list(counts)
    if rc == -2:
        raise CapacityError(f"row segments need {sum(out)} rows > capacity {rows_cap}", counts=out,
                            needed=sum(out), rows_cap=rows_cap)
    if rc != 0:
        raise nat.NativeError(f"mgb_moe_check_capacity failed: {nat.STATUS.get(rc, rc)}")
    return out


SITES = {1: "moe_gemm_gate_up", 2: "moe_gemm_down", 3: "ep_permute_dispatch"}


def capacity_status(reset: bool = True) -> None:
    """Raise CapacityError if a grouped GEMM / EP dispatch recorded an overflow on this device since
    the last call (synchronises the device; cleared when reset)."""
    import ctypes

    st = (ctypes.c_int * 4)()
    rc = nat.raw("mgb_capacity_status", st, int(reset))
    if rc == -2:
        raise CapacityError(f"{SITES.get(st[3], st[3])}: {st[1]} rows needed > capacity {st[2]} (no rows were "
                            f"written past the buffer)", needed=st[1], rows_cap=st[2], site=st[3])
    if rc != 0:
        raise nat.NativeError(f"mgb_capacity_status failed: {nat.STATUS.get(rc, rc)}")


def moe_gemm_gate_up(w_gate_up: torch.Tensor, x_perm: torch.Tensor, offsets: torch.Tensor, h_out: torch.Tensor) -> None:
    E, two_f, d = w_gate_up.shape
    nat.call("mgb_moe_gemm_gate_up", _p(w_gate_up), _p(x_perm), _p(offsets), E, d, two_f // 2, x_perm.shape[0],
             _p(h_out), _s())


def moe_gemm_down(w_down: torch.Tensor, h: torch.Tensor, offsets: torch.Tensor, y_out: torch.Tensor) -> None:
    E, d, f = w_down.shape
    nat.call("mgb_moe_gemm_down", _p(w_down), _p(h), _p(offsets), E, d, f, h.shape[0], _p(y_out), _s())


def moe_ffn(w_gate_up: torch.Tensor, w_down: torch.Tensor, x_perm: torch.Tensor, offsets: torch.Tensor,
            h: torch.Tensor, y_out: torch.Tensor, sync: torch.Tensor) -> None:
    """The whole grouped expert FFN in one launch (gate/up + SiLU*up + down; mgb_moe_ffn).
    sync: int32 [257] zeros, reused across launches (each launch leaves it zero)."""
    E, two_f, d = w_gate_up.shape
    assert sync.numel() >= 257 and sync.dtype == torch.int32
    nat.call("mgb_moe_ffn", _p(w_gate_up), _p(w_down), _p(x_perm), _p(offsets), E, d, two_f // 2, x_perm.shape[0],
             _p(h), _p(y_out), _p(sync), _s())


def unpermute_combine(y_perm: torch.Tensor, ws: RouterWorkspace, out: torch.Tensor, T: int,
                      residual: torch.Tensor | None = None, shared_out: torch.Tensor | None = None,
                      norm_w: torch.Tensor | None = None, eps: float = 0.0,
                      norm_out: torch.Tensor | None = None) -> None:
    nat.call("mgb_unpermute_combine", _p(y_perm), _p(ws.dst_pos), _p(ws.topk_w), _p(shared_out), _p(residual), T,
             out.shape[1], ws.k, _p(out), _p(norm_w), eps, _p(norm_out), _s())


def add_rmsnorm(x: torch.Tensor, weight: torch.Tensor, eps: float, y: torch.Tensor,
                delta: torch.Tensor | None = None, x_out: torch.Tensor | None = None) -> None:
    T, d = x.shape
    nat.call("mgb_add_rmsnorm", _p(x), _p(delta), _p(weight), eps, T, d, _p(x_out), _p(y), _s())


def rope_append_gqa(qkv: torch.Tensor, seq0: int, positions: torch.Tensor, cos_t: torch.Tensor, sin_t: torch.Tensor,
                    Hq: int, Hkv: int, hd: int, block_table: torch.Tensor, k_cache: torch.Tensor,
                    v_cache: torch.Tensor, q_out: torch.Tensor, seq_lens: torch.Tensor | None = None) -> None:
    T = qkv.shape[0]
    nat.call("mgb_rope_append_gqa", _p(qkv), T, seq0, _p(positions), _p(cos_t), _p(sin_t), Hq, Hkv, hd,
             _p(block_table), block_table.shape[1], _p(k_cache), _p(v_cache), _p(q_out), _p(seq_lens), _s())


def decode_attn_gqa(q: torch.Tensor, k_cache: torch.Tensor, v_cache: torch.Tensor, block_table: torch.Tensor,
                    seq_lens: torch.Tensor, Hq: int, Hkv: int, hd: int, out: torch.Tensor,
                    scale: float | None = None, sched: torch.Tensor | None = None) -> None:
    """sched: int32 [2] zeros (reused; launches sharing it must be stream-ordered) -> dynamic item
    scheduling across the persistent CTAs; None -> the static round-robin share."""
    B = q.shape[0]
    scale = hd ** -0.5 if scale is None else scale
    if sched is None:
        nat.call("mgb_decode_attn_gqa", _p(q), _p(k_cache), _p(v_cache), _p(block_table), block_table.shape[1],
                 _p(seq_lens), B, Hq, Hkv, hd, scale, _p(out), _s())
    else:
        nat.call("mgb_decode_attn_gqa_sched", _p(q), _p(k_cache), _p(v_cache), _p(block_table), block_table.shape[1],
                 _p(seq_lens), B, Hq, Hkv, hd, scale, _p(out), _p(sched), _s())


def decode_attn_gqa_rope(qkv: torch.Tensor, positions: torch.Tensor, cos_t: torch.Tensor, sin_t: torch.Tensor,
                         k_cache: torch.Tensor, v_cache: torch.Tensor, block_table: torch.Tensor,
                         seq_lens: torch.Tensor, Hq: int, Hkv: int, hd: int, out: torch.Tensor,
                         scale: float | None = None, sched: torch.Tensor | None = None) -> None:
    """Decode attention with the step's RoPE + KV append fused in: qkv [B, (Hq + 2 Hkv) hd] raw
    projections, positions [B]; appends the rotated k / the v row at each position, writes
    seq_lens = positions + 1 and out = attention over positions 0..pos (= rope_append_gqa followed by
    decode_attn_gqa, bit-identical)."""
    B = qkv.shape[0]
    scale = hd ** -0.5 if scale is None else scale
    nat.call("mgb_decode_attn_gqa_rope", _p(qkv), _p(positions), _p(cos_t), _p(sin_t), _p(k_cache), _p(v_cache),
             _p(block_table), block_table.shape[1], _p(seq_lens), B, Hq, Hkv, hd, scale, _p(out), _p(sched), _s())


def prefill_attn_supported(hd_qk: int, hd_v: int) -> bool:
    return bool(nat.value("mgb_prefill_attn_supported", hd_qk, hd_v))


def prefill_attn(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor, n_seq: int, P: int, Hq: int,
                 Hkv: int, hd_qk: int, hd_v: int, scale: float, q_head_cols: int, k_head_cols: int, v_head_cols: int,
                 v_col0: int = 0, kr: torch.Tensor | None = None) -> None:
    """Causal prefill attention (tcgen05, attn_prefill.cu) over 2-D row-major [n_seq*P, cols] tensors;
    `kr` holds MLA's shared rope part of K (its width is the last kr.shape[1] dims of hd_qk)."""
    for t in (q, k, v, out) + ((kr,) if kr is not None else ()):
        assert t.dim() == 2 and t.stride(1) == 1 and t.dtype == BF16
    kr_cols = kr.stride(0) if kr is not None else 0
    kr_dim = kr.shape[1] if kr is not None else 0
    nat.call("mgb_prefill_attn", _p(q), q.stride(0), q_head_cols, _p(k), k.stride(0), k_head_cols, _p(kr), kr_cols,
             kr_dim, _p(v), v.stride(0), v_head_cols, v_col0, n_seq, P, Hq, Hkv, hd_qk, hd_v, scale, _p(out),
             out.stride(0), _s())


def silu_mul(gate_up: torch.Tensor, h: torch.Tensor) -> None:
    T, F = h.shape
    assert gate_up.shape == (T, 2 * F) and gate_up.is_contiguous() and h.is_contiguous()
    nat.call("mgb_silu_mul", _p(gate_up), T, F, _p(h), _s())


def embed(ids: torch.Tensor, table: torch.Tensor, out: torch.Tensor) -> None:
    nat.call("mgb_embed", _p(ids), _p(table), ids.shape[0], table.shape[1], _p(out), _s())


def argmax(logits: torch.Tensor, out: torch.Tensor) -> None:
    T, V = logits.shape
    nat.call("mgb_argmax", _p(logits), T, V, _p(out), _s())


def decode_advance(next_ids: torch.Tensor, out_tokens: torch.Tensor | None, step: torch.Tensor,
                   positions: torch.Tensor) -> None:
    B = next_ids.shape[0]
    ld = out_tokens.shape[1] if out_tokens is not None else 0
    nat.call("mgb_decode_advance", _p(next_ids), B, _p(out_tokens), ld, _p(step), _p(positions), _s())


def kv_page_size() -> int:
    return nat.value("mgb_kv_page_size")
