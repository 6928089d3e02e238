"""Shared parity machinery for the engine-vs-oracle GPU tests (test infrastructure only).

`layer_parity` drives one decode position through the engine layer by layer (the engine's own job
issue, `Engine._issue_layer`) next to the CPU oracle, re-synchronising the residual stream to the
oracle after every layer, and applies the north_star bar per layer (BASELINE.json: "max relative
error 2e-2 per layer"):

  - routing: the engine's top-k indices are bit-exact vs the oracle router run on the engine's own
    router logits; where the engine-vs-oracle expert sets (each side routing
    its own hidden state) differ, the oracle's k-th / (k+1)-th router logit gap is within 4x the
    largest router-logit difference (a near-tie; greedy modes), and at most max(2, B/50) rows
    of a layer differ;
  - every row: attention output and router input h2 within max|a-b|/max|b| <= 2e-2;
  - every row whose routing matches the oracle's: the layer output row within 2e-2.  A row whose
    near-tied bf16 router logit picked another expert is reported, not failed.
"""

from __future__ import annotations

import torch

from oracle import moe_ref as R

TOL = 2e-2


def oracle_weights(eng) -> R.MixtralWeights:
    """The engine's weights in the oracle's layout (CPU copies)."""
    a, w = eng.arch, eng.w
    layers = []
    for L in w.layers:
        c = {k: v.cpu() for k, v in L.items() if k not in ("w_uk", "w_uv_t") and v is not None}
        if a.family == "mixtral":
            hd = a.head_dim
            qd, kvd = a.n_heads * hd, a.n_kv_heads * hd
            wqkv = c.pop("wqkv")
            c.update(wq=wqkv[:qd], wk=wqkv[qd:qd + kvd], wv=wqkv[qd + kvd:])
        else:
            for k in ("sh_gate_up", "sh_down", "dense_gate_up", "dense_down"):
                if k in c:
                    c[k] = c[k][0]
        layers.append(c)
    return R.MixtralWeights(embed=w.embed.cpu(), final_norm=w.final_norm.cpu(), lm_head=w.lm_head.cpu(),
                            layers=layers)


def gqa_pages_to_dense(store: torch.Tensor, B: int, pps: int, Hkv: int, hd: int, page: int, ctx: int):
    """Engine GQA page store (pages [Hkv][hd/8][page][8], identity block table) -> [B, Hkv, ctx, hd]."""
    x = store.cpu().view(B, pps, Hkv, hd // 8, page, 8).permute(0, 2, 1, 4, 3, 5)
    return x.reshape(B, Hkv, pps * page, hd)[:, :, :ctx].contiguous()


def mla_pages_to_dense(store: torch.Tensor, B: int, pps: int, page: int, R_: int, r: int, ctx: int):
    """Engine latent page store ([ceil(D/64)][page][64] per page, 16-byte chunk j of token t stored at
    j ^ (t % 8), attn_mla.cu) -> (c [B, ctx, R], k_pe [B, ctx, r])."""
    D = R_ + r
    nkb = (D + 63) // 64
    x = store.cpu().view(B, pps, nkb, page, 8, 8)
    t = torch.arange(page)
    src = torch.arange(8)[None, :] ^ (t[:, None] % 8)          # logical chunk c of token t is stored at c ^ (t%8)
    x = x[:, :, :, t[:, None], src, :]                          # [B, pps, nkb, page, 8(c), 8]
    x = x.permute(0, 1, 3, 2, 4, 5).reshape(B, pps * page, nkb * 64)[:, :ctx, :D]
    return x[..., :R_].contiguous(), x[..., R_:].contiguous()


def load_oracle_kv(eng, orc, ctx: int) -> None:
    """Hand the engine's first `ctx` cached positions of every layer to the oracle (the synthetic
    prefill state the bench decodes from)."""
    a = eng.arch
    for l in range(a.layers):
        if eng.mla:
            c, pe = mla_pages_to_dense(eng.latent[l], eng.B, eng.pps, eng.page, a.kv_lora_rank, a.qk_rope_dim, ctx)
            orc.set_latent(l, c, pe)
        else:
            k = gqa_pages_to_dense(eng.k_cache[l], eng.B, eng.pps, a.n_kv_heads, a.head_dim, eng.page, ctx)
            v = gqa_pages_to_dense(eng.v_cache[l], eng.B, eng.pps, a.n_kv_heads, a.head_dim, eng.page, ctx)
            orc.set_kv(l, k, v)


def row_errs(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """Per-row max|a-b| / max|b| (the north_star per-layer metric, row by row)."""
    a, b = a.float(), b.float()
    return (a - b).abs().amax(-1) / b.abs().amax(-1).clamp_min(1e-30)


def _router_logits_engine(eng, l: int) -> torch.Tensor:
    """The fp32 router logits the engine's router kernel consumed for layer l (as the kernel sees
    them: Mixtral rounds them to bf16 first, as HF's bf16 gate does, modeling_mixtral.py:111)."""
    if eng.mla:
        return eng.mb["logits_r"].cpu()
    return eng.logits_r.cpu().to(torch.bfloat16).float()


def layer_parity(eng, orc, tokens: torch.Tensor, pos: int, report: dict | None = None):
    """One decode position, layer by layer, re-synchronised; asserts the per-layer bar and returns
    (engine logits, oracle logits), fp32 CPU, each side from its own last-layer output."""
    from paper_2503_09716_b200 import ops

    a, b = eng.arch, eng.buf
    B = tokens.shape[0]
    b.positions.fill_(pos)
    b.next_ids.copy_(tokens.to(torch.int32))
    ops.embed(b.next_ids, eng.w.embed, b.x)
    x = orc.w.embed[tokens]
    assert torch.equal(b.x.cpu(), x)
    logits_e = None
    for l in range(a.layers):
        tr = {}
        x = orc.layer_forward(l, x, pos, tr)
        eng.debug_taps = {}
        torch.cuda.synchronize()  # the embed / re-sync writes (current stream) land before the engine stream reads
        with torch.cuda.stream(eng.stream):
            eng._issue_layer(l)
        torch.cuda.synchronize()
        taps, eng.debug_taps = eng.debug_taps, None
        attn_e = (eng.mb["o_cat"] if eng.mla else b.attn).cpu()
        e_attn = row_errs(attn_e, tr["attn"])
        assert e_attn.max() <= TOL, f"layer {l}: attention row err {e_attn.max():.3e}"
        e_x = row_errs(b.x.cpu(), x)
        moe = "topk_idx" in taps
        if moe:
            e_h2 = row_errs(taps["h2"].cpu(), tr["h2"])
            assert e_h2.max() <= TOL, f"layer {l}: router input row err {e_h2.max():.3e}"
            idx_e = taps["topk_idx"].cpu().long()
            # bit-exact given identical logits
            lg = _router_logits_engine(eng, l)
            idx_r, _ = R.route(lg, a.top_k, a.router_mode, a.routed_scaling, a.n_group, a.topk_group)
            assert torch.equal(idx_r, idx_e), f"layer {l}: router indices differ from the oracle on the same logits"
            match = (idx_e.sort(-1).values == tr["topk_idx"].sort(-1).values).all(-1)
            agree = match.float().mean().item()
            n_bad = int((~match).sum())
            # sanity bound; the real bar is the near-tie explanation below (a flip needs a near-tied
            # k-th / (k+1)-th router logit)
            assert n_bad <= max(2, B // 50), f"layer {l}: routing agreement {agree:.4f}"
            if n_bad and a.router_mode != 2:
                # every disagreement must be a near-tie: the oracle's k-th / (k+1)-th logit gap is
                # within 4x the largest engine-vs-oracle router-logit difference
                lo_r = tr["logits"].float()
                delta = (lg - lo_r).abs().max().item()
                srt = lo_r[~match].sort(-1, descending=True).values
                gap = srt[:, a.top_k - 1] - srt[:, a.top_k]
                assert bool((gap <= 4 * delta).all()), f"layer {l}: routing differs on a row without a near-tie"
        else:
            match = torch.ones(B, dtype=torch.bool)
            agree = 1.0
        worst = e_x[match].max().item()
        assert worst <= TOL, f"layer {l}: worst routing-matched row err {worst:.3e}"
        if report is not None:
            report.setdefault("layers", []).append(dict(
                layer=l, pos=pos, attn_max=float(e_attn.max()), x_max_matched=worst,
                x_max_all=float(e_x.max()), routing_agreement=agree, rows=B, mismatched_rows=int((~match).sum())))
        if l == a.layers - 1:  # logits from the engine's own last-layer output (fused final norm)
            logits_e = torch.mm(b.h, eng.w.lm_head.t()).float().cpu()
        b.x.copy_(x)  # re-synchronise the residual stream (and the fused next-layer norm)
        nxt = eng.w.layers[l + 1]["ln1"] if l + 1 < a.layers else eng.w.final_norm
        ops.add_rmsnorm(b.x, nxt, a.rms_eps, b.h)
    torch.cuda.synchronize()
    return logits_e, oracle_logits(orc, x)


def oracle_logits(orc, x_last: torch.Tensor) -> torch.Tensor:
    a = orc.a
    return torch.nn.functional.linear(R.rmsnorm(x_last, orc.w.final_norm, a.rms_eps), orc.w.lm_head).float()


def margin_filtered_equal(le: torch.Tensor, lo: torch.Tensor) -> tuple[bool, int]:
    """Greedy argmax identical on every row whose oracle top1-top2 margin exceeds 4x the largest
    |delta logit|; returns (ok, rows checked)."""
    delta = (le - lo).abs().max().item()
    top2 = lo.topk(2, dim=-1).values
    safe = (top2[:, 0] - top2[:, 1]) > 4 * delta
    return bool(torch.equal(le.argmax(-1)[safe], lo.argmax(-1)[safe])), int(safe.sum())


def greedy_prefix(out: torch.Tensor, ref: torch.Tensor, P: int) -> torch.Tensor:
    """Per row: number of leading generated tokens identical to the reference (unfiltered)."""
    gen_e, gen_r = out[:, P:], ref[:, P:]
    diff = (gen_e != gen_r)
    n = gen_e.shape[1]
    first = torch.where(diff.any(1), diff.float().argmax(1), torch.full((out.shape[0],), n))
    return first
