"""GPU parity of every libmgb kernel against the CPU oracle (oracle/moe_ref.py) on seeded inputs.

Bars (BASELINE.json north_star): routing indices and permutations bit-exact given identical
logits; integer/byte outputs bit-exact; bf16 arithmetic within the stated tolerance."""

import math

import pytest
import torch

from oracle import moe_ref as R
from oracle.rng import uniform_bf16

pytestmark = pytest.mark.gpu

BF16 = torch.bfloat16


def _ops():
    from paper_2503_09716_b200 import ops

    return ops


@pytest.mark.parametrize("T,E,k,mode,ng,tg", [
    (1, 8, 2, 0, 1, 1), (64, 8, 2, 0, 1, 1), (777, 8, 2, 0, 1, 1), (300, 64, 6, 1, 1, 1),
    (257, 160, 6, 2, 8, 3), (40, 16, 4, 2, 4, 2), (1024, 64, 6, 1, 1, 1), (6058, 64, 6, 1, 1, 1),
    (3001, 160, 6, 2, 8, 3), (9000, 8, 2, 0, 1, 1)])
def test_router_topk_bitexact_given_logits(T, E, k, mode, ng, tg):
    ops = _ops()
    g = torch.Generator().manual_seed(T * 31 + E)
    logits = torch.randn(T, E, generator=g)
    # force exact ties to exercise the pinned tie rule
    logits[:, 1] = logits[:, 0]
    logits = logits.to(BF16).float() if mode == 0 else logits
    ws = ops.RouterWorkspace(T, E, k)
    ops.router_topk(None, None, ws, k, mode, 2.5, ng, tg, logits_in=logits.cuda())
    idx_ref, w_ref = R.route(logits, k, mode, 2.5, ng, tg)
    assert torch.equal(ws.topk_idx.cpu().long(), idx_ref)
    torch.testing.assert_close(ws.topk_w.cpu(), w_ref.float(), rtol=2e-6, atol=1e-7)
    order, dst, counts, offsets = R.permutation(idx_ref, E)
    assert torch.equal(ws.counts.cpu().long(), counts)
    assert torch.equal(ws.offsets.cpu().long(), offsets)
    # the ticket self-resets (graph-replay safe)
    assert int(ws.ticket.item()) == 0


def test_router_workspace_serves_smaller_batches():
    """One workspace sized for 6058 tokens routes micro-batches of other sizes in turn (histograms,
    ticket and offsets reused; the ticket self-resets between calls)."""
    ops = _ops()
    ws = ops.RouterWorkspace(6058, 64, 6)
    for T in (2000, 6058, 5):
        logits = torch.randn(T, 64, generator=torch.Generator().manual_seed(T))
        ops.router_topk(None, None, ws, 6, 1, 1.0, logits_in=logits.cuda())
        idx_ref, _ = R.route(logits, 6, 1, 1.0)
        assert torch.equal(ws.topk_idx[:T].cpu().long(), idx_ref)
        _, _, counts, offsets = R.permutation(idx_ref, 64)
        assert torch.equal(ws.offsets.cpu().long(), offsets)


@pytest.mark.parametrize("T,d,E,k,mode", [(64, 256, 8, 2, 0), (513, 4096, 8, 2, 0), (200, 2048, 64, 6, 1),
                                          (3001, 1024, 64, 6, 1)])
def test_router_gemv_and_permutation(T, d, E, k, mode):
    ops = _ops()
    x = uniform_bf16((T, d), 3, 7, 1.0)
    wg = uniform_bf16((E, d), 3, 8, 0.02)
    ws = ops.RouterWorkspace(T, E, k)
    logits_out = torch.zeros(T, E, device="cuda")
    ops.router_topk(x.cuda(), wg.cuda(), ws, k, mode, logits_out=logits_out)
    lg = logits_out.cpu()
    # logits: fp32 accumulation of bf16 products (+ bf16 rounding for Mixtral)
    ref = torch.nn.functional.linear(x.float(), wg.float())
    if mode == 0:
        ref = ref.to(BF16).float()
    assert (lg - ref).abs().max().item() <= (1e-2 if mode == 0 else 1e-4) * ref.abs().max().item()
    # routing from the kernel's own logits is bit-exact vs the oracle
    idx_ref, w_ref = R.route(lg, k, mode)
    assert torch.equal(ws.topk_idx.cpu().long(), idx_ref)
    # permutation: bit-exact stable expert-major order + gathered rows
    x_perm = torch.zeros(T * k, d, dtype=BF16, device="cuda")
    ops.permute(x.cuda(), ws, x_perm)
    order, dst, counts, offsets = R.permutation(idx_ref, E)
    assert torch.equal(ws.dst_pos.cpu().long(), dst)
    assert torch.equal(ws.src_token.cpu().long(), order // k)
    assert torch.equal(x_perm.cpu(), x[order // k])


def _ffn_ref(x_perm, offsets, wgu, wd):
    rows, d = x_perm.shape
    E = wgu.shape[0]
    out = torch.zeros(rows, d, dtype=BF16)
    for e in range(E):
        a, b = int(offsets[e]), int(offsets[e + 1])
        if b > a:
            out[a:b] = R.expert_ffn(x_perm[a:b], wgu[e], wd[e])
    return out


@pytest.mark.parametrize("E,d,f,counts", [
    (8, 256, 512, [0, 1, 17, 33, 64, 100, 255, 300]),
    (4, 512, 384, [256, 257, 512, 3]),
    (16, 256, 128, [5] * 16),
    (2, 1024, 1024, [600, 0])])
def test_grouped_ffn_tcgen05(E, d, f, counts):
    ops = _ops()
    offs = [0]
    for c in counts:
        offs.append(offs[-1] + c)
    rows = offs[-1]
    x = uniform_bf16((rows, d), 5, 1, 1.0)
    wgu = uniform_bf16((E, 2 * f, d), 5, 2, 0.05)
    wd = uniform_bf16((E, d, f), 5, 3, 0.05)
    offsets = torch.tensor(offs, dtype=torch.int32)
    H = torch.zeros(rows, f, dtype=BF16, device="cuda")
    Y = torch.zeros(rows, d, dtype=BF16, device="cuda")
    ops.moe_gemm_gate_up(wgu.cuda(), x.cuda(), offsets.cuda(), H)
    ops.moe_gemm_down(wd.cuda(), H, offsets.cuda(), Y)
    ref = _ffn_ref(x, offsets, wgu, wd)
    # tolerance: fp32 accumulation order differs from the CPU GEMM; bf16 outputs
    assert R.rel_err(Y.cpu(), ref) <= 2e-2
    assert R.cosine(Y.cpu(), ref) >= 0.9999


@pytest.mark.parametrize("T,d,k", [(5, 256, 2), (300, 4096, 2), (64, 2048, 6)])
def test_unpermute_combine(T, d, k):
    ops = _ops()
    E = 8
    g = torch.Generator().manual_seed(T)
    logits = torch.randn(T, E, generator=g)
    idx, w = R.route(logits, k, 0)
    order, dst, counts, offsets = R.permutation(idx, E)
    y = uniform_bf16((T * k, d), 9, 1, 1.0)
    res = uniform_bf16((T, d), 9, 2, 1.0)
    ws = ops.RouterWorkspace(T, E, k)
    ws.dst_pos.copy_(dst.to(torch.int32))
    ws.topk_w.copy_(w)
    out = torch.zeros(T, d, dtype=BF16, device="cuda")
    ops.unpermute_combine(y.cuda(), ws, out, T, residual=res.cuda())
    acc = torch.zeros(T, d)
    for j in range(k):
        acc += y[dst.view(T, k)[:, j]].float() * w[:, j:j + 1]
    ref = res + acc.to(BF16)
    # k=2: the fp32 sum is order independent -> bit-exact; k=6: ulp-level
    if k == 2:
        assert torch.equal(out.cpu(), ref)
    else:
        assert R.rel_err(out.cpu(), ref) <= 1e-2


def test_fill_uniform_matches_oracle_rng():
    from paper_2503_09716_b200.weights import fill_uniform_

    t = torch.empty(3, 1000, dtype=BF16, device="cuda")
    fill_uniform_(t, 7, 12345, 0.02)
    assert torch.equal(t.cpu(), uniform_bf16((3, 1000), 7, 12345, 0.02))


def test_add_rmsnorm():
    ops = _ops()
    T, d = 37, 4096
    x = uniform_bf16((T, d), 2, 1, 1.0)
    dl = uniform_bf16((T, d), 2, 2, 1.0)
    w = uniform_bf16((d,), 2, 3, 1.0)
    xo = x.cuda().clone()
    y = torch.zeros(T, d, dtype=BF16, device="cuda")
    ops.add_rmsnorm(xo, w.cuda(), 1e-5, y, delta=dl.cuda(), x_out=xo)
    xs = x + dl
    assert torch.equal(xo.cpu(), xs)
    ref = R.rmsnorm(xs, w, 1e-5)
    assert R.rel_err(y.cpu(), ref) <= 1e-2


def _paged_kv(kc, vc, B, Hkv, hd, ctx, page, pps, tail=0.0):
    """dense [B,Hkv,ctx,hd] -> engine page layout (K and V chunk-major [hd/8][page][8]); rows past
    ctx hold `tail` (the kernel must ignore them, NaN / Inf included)."""
    kp = torch.full((B * pps, Hkv, hd // 8, page, 8), tail, dtype=BF16)
    vp = torch.full((B * pps, Hkv, hd // 8, page, 8), tail, dtype=BF16)
    for b in range(B):
        for t in range(ctx):
            pg, s = b * pps + t // page, t % page
            kp[pg, :, :, s, :] = kc[b, :, t, :].view(Hkv, hd // 8, 8)
            vp[pg, :, :, s, :] = vc[b, :, t, :].view(Hkv, hd // 8, 8)
    return kp.reshape(-1), vp.reshape(-1)


@pytest.mark.parametrize("B,Hq,Hkv,hd,ctx,tail", [(3, 32, 8, 128, 1, 0.0), (5, 32, 8, 128, 200, 0.0),
                                                  (4, 8, 2, 32, 130, 0.0), (2, 48, 8, 128, 64, 0.0),
                                                  (3, 32, 8, 128, 70, float("nan")), (2, 32, 8, 128, 17, float("inf")),
                                                  (4, 8, 2, 32, 100, float("nan"))])
def test_decode_attn_gqa(B, Hq, Hkv, hd, ctx, tail):
    ops = _ops()
    page = ops.kv_page_size()
    pps = math.ceil(ctx / page)
    q = uniform_bf16((B, Hq, hd), 4, 1, 1.0)
    kc = uniform_bf16((B, Hkv, ctx, hd), 4, 2, 1.0)
    vc = uniform_bf16((B, Hkv, ctx, hd), 4, 3, 1.0)
    kp, vp = _paged_kv(kc, vc, B, Hkv, hd, ctx, page, pps, tail)
    bt = torch.arange(B * pps, dtype=torch.int32).view(B, pps)
    lens = torch.full((B,), ctx, dtype=torch.int32)
    out = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
    ops.decode_attn_gqa(q.cuda(), kp.cuda(), vp.cuda(), bt.cuda(), lens.cuda(), Hq, Hkv, hd, out)
    ref = R.gqa_decode_attention(q, kc, vc)  # sdpa semantics: fp32 inside, one bf16 rounding
    eager = R.gqa_decode_attention(q, kc, vc, impl="eager")
    assert R.rel_err(out.cpu(), ref) <= 1e-2
    assert R.rel_err(out.cpu(), eager) <= 2e-2


@pytest.mark.parametrize("B,ctx", [(3, 200), (600, 70), (2000, 33)])
def test_decode_attn_gqa_dynamic_schedule(B, ctx):
    """Dynamic item scheduling (mgb_decode_attn_gqa_sched) gives the static kernel's output bit for bit
    (every item is computed the same way, only its CTA changes) and leaves its counters at zero."""
    ops = _ops()
    Hq, Hkv, hd = 32, 8, 128
    page = ops.kv_page_size()
    pps = math.ceil(ctx / page)
    q = uniform_bf16((B, Hq, hd), 6, 1, 1.0).cuda()
    kp = uniform_bf16((B * pps * Hkv * hd * page,), 6, 2, 1.0).cuda()
    vp = uniform_bf16((B * pps * Hkv * hd * page,), 6, 3, 1.0).cuda()
    bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
    lens = torch.randint(1, ctx + 1, (B,), generator=torch.Generator().manual_seed(B)).int().cuda()
    ref = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
    ops.decode_attn_gqa(q, kp, vp, bt, lens, Hq, Hkv, hd, ref)
    sched = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(3):
        out = torch.zeros_like(ref)
        ops.decode_attn_gqa(q, kp, vp, bt, lens, Hq, Hkv, hd, out, sched=sched)
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        assert int(sched.abs().sum()) == 0


@pytest.mark.parametrize("B", [3, 301, 1001])  # 301 / 1001: several tokens per CTA (decode batches)
def test_rope_append_matches_oracle(B):
    ops = _ops()
    Hq, Hkv, hd, pos = 8, 2, 32, 70
    page = ops.kv_page_size()
    pps = 2
    qkv = uniform_bf16((B, (Hq + 2 * Hkv) * hd), 6, 1, 1.0)
    theta = 1e6
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    fr = torch.arange(128).float()[:, None] * inv[None]
    cos_t, sin_t = fr.cos().to(BF16).float(), fr.sin().to(BF16).float()
    kc = torch.zeros(B * pps * Hkv * hd * page, dtype=BF16, device="cuda")
    vc = torch.zeros_like(kc)
    qo = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
    bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
    pos_h = pos + torch.arange(B, dtype=torch.int32) % 7  # ragged: pages 1, slots 6..12
    positions = pos_h.cuda()
    lens = torch.zeros(B, dtype=torch.int32, device="cuda")
    ops.rope_append_gqa(qkv.cuda(), 0, positions, cos_t.cuda(), sin_t.cuda(), Hq, Hkv, hd, bt, kc, vc, qo, lens)
    cos, sin = R.rope_cos_sin(theta, hd, pos_h.long())
    q = qkv[:, :Hq * hd].view(B, Hq, hd)
    k = qkv[:, Hq * hd:(Hq + Hkv) * hd].view(B, Hkv, hd)
    v = qkv[:, (Hq + Hkv) * hd:].view(B, Hkv, hd)
    assert torch.equal(qo.cpu().view(B, Hq, hd), R.apply_rope(q, cos, sin))
    kref = R.apply_rope(k, cos, sin)
    kp = kc.cpu().view(B * pps, Hkv, hd // 8, page, 8)
    vp = vc.cpu().view(B * pps, Hkv, hd // 8, page, 8)
    for b in range(B):
        pb = int(pos_h[b])
        pg, s = b * pps + pb // page, pb % page
        assert torch.equal(kp[pg, :, :, s, :].reshape(Hkv, hd), kref[b])
        assert torch.equal(vp[pg, :, :, s, :].reshape(Hkv, hd), v[b])
    assert torch.equal(lens.cpu(), pos_h + 1)


@pytest.mark.parametrize("B,Hq,Hkv,hd", [(37, 32, 8, 128), (300, 32, 8, 128), (9, 8, 2, 32), (5, 16, 4, 64)])
def test_decode_attn_gqa_rope_fused_matches_two_launches(B, Hq, Hkv, hd):
    """mgb_decode_attn_gqa_rope (RoPE + KV append inside the attention launch) against
    mgb_rope_append_gqa followed by mgb_decode_attn_gqa_sched on copies of the same cache: ragged
    positions (first slot of a page, page boundaries, the last planned slot), pages holding garbage
    past each sequence's end -> identical attention output, K / V pages and seq_lens, bit for bit."""
    ops = _ops()
    page = ops.kv_page_size()
    pps = 5
    g = torch.Generator().manual_seed(B + hd)
    positions = torch.randint(0, pps * page, (B,), generator=g, dtype=torch.int32)
    positions[:4] = torch.tensor([0, page, page - 1, pps * page - 1], dtype=torch.int32)[:min(4, B)]
    qkv = uniform_bf16((B, (Hq + 2 * Hkv) * hd), 9, B, 1.0).cuda()
    theta = 1e6
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.int64).float() / hd))
    fr = torch.arange(pps * page).float()[:, None] * inv[None]
    cos_t, sin_t = fr.cos().to(BF16).float().cuda(), fr.sin().to(BF16).float().cuda()
    kc = uniform_bf16((B * pps * Hkv * hd * page,), 10, B, 1.0).cuda()
    vc = uniform_bf16((B * pps * Hkv * hd * page,), 11, B, 1.0).cuda()
    perm = torch.randperm(B * pps, generator=g).to(torch.int32)
    bt = perm.view(B, pps).cuda()
    pos_d = positions.cuda()
    # two launches
    k1, v1 = kc.clone(), vc.clone()
    q1 = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
    lens1 = torch.zeros(B, dtype=torch.int32, device="cuda")
    out1 = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
    ops.rope_append_gqa(qkv, 0, pos_d, cos_t, sin_t, Hq, Hkv, hd, bt, k1, v1, q1, lens1)
    ops.decode_attn_gqa(q1, k1, v1, bt, lens1, Hq, Hkv, hd, out1, sched=torch.zeros(2, dtype=torch.int32, device="cuda"))
    # fused, twice (the scheduler counter returns to zero)
    sched = torch.zeros(2, dtype=torch.int32, device="cuda")
    for _ in range(2):
        k2, v2 = kc.clone(), vc.clone()
        lens2 = torch.zeros(B, dtype=torch.int32, device="cuda")
        out2 = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
        ops.decode_attn_gqa_rope(qkv, pos_d, cos_t, sin_t, k2, v2, bt, lens2, Hq, Hkv, hd, out2, sched=sched)
    torch.cuda.synchronize()
    assert torch.equal(lens2, lens1) and torch.equal(lens1.cpu(), positions + 1)
    assert torch.equal(k2, k1) and torch.equal(v2, v1)
    assert torch.equal(out2, out1)
    assert int(sched.abs().sum()) == 0


def test_argmax_first_index():
    ops = _ops()
    lg = torch.randn(9, 32000).to(BF16)
    lg[3, 100] = lg[3, 200] = 50.0
    out = torch.zeros(9, dtype=torch.int32, device="cuda")
    ops.argmax(lg.cuda(), out)
    assert torch.equal(out.cpu().long(), torch.argmax(lg.float(), dim=-1))
