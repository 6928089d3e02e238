"""Small launches of every libmgb kernel family for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): router, fused route, permute, grouped GEMMs, fused FFN, combine, GQA / MLA
decode attention, RoPE / latent append, prefill attention.  Eager, tiny shapes, no graphs.

compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.rng import uniform_bf16  # noqa: E402
from paper_2503_09716_b200 import _native as nat  # noqa: E402
from paper_2503_09716_b200 import ops  # noqa: E402

BF = torch.bfloat16
dev = "cuda"
st = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731

# routing + permutation + grouped FFN + combine (Mixtral-like, small)
T, d, f, E, k = 40, 256, 512, 8, 2
x = uniform_bf16((T, d), 0, 1, 1.0).to(dev)
o = uniform_bf16((T, d), 0, 2, 1.0).to(dev)
ln = torch.ones(d, dtype=BF, device=dev)
wr = uniform_bf16((E, d), 0, 3, 0.1).to(dev)
wgu = uniform_bf16((E, 2 * f, d), 0, 4, 0.05).to(dev)
wd = uniform_bf16((E, d, f), 0, 5, 0.05).to(dev)
ws = ops.RouterWorkspace(T, E, k)
h = torch.zeros(T, d, dtype=BF, device=dev)
xp = torch.zeros(T * k, d, dtype=BF, device=dev)
ops.moe_route(x, o, ln, 1e-5, h, wr, ws, xp, 0, x_out=torch.zeros_like(x))
ops.moe_route(x, o, ln, 1e-5, None, wr, ops.RouterWorkspace(T, E, k), torch.zeros_like(xp), 0,
              x_out=torch.zeros_like(x))  # one pass without h_out (decode batches)
# > 1 chunk per CTA (rows re-read from h_out) on a wider batch
T2 = 3001
x2 = uniform_bf16((T2, d), 0, 6, 1.0).to(dev)
ops.moe_route(x2, None, ln, 1e-5, torch.zeros_like(x2), wr, ops.RouterWorkspace(T2, E, k),
              torch.zeros(T2 * k, d, dtype=BF, device=dev), 0)
# DeepSeek-width router over given logits (many CTAs: separate column scan)
lg2 = torch.randn(T2, 64, device=dev)
ops.router_topk(None, None, ops.RouterWorkspace(T2, 64, 6), 6, 1, logits_in=lg2)
# an expert-parallel rank's weight shard generated in place
from paper_2503_09716_b200.weights import fill_uniform_  # noqa: E402
fill_uniform_(torch.empty(4097, dtype=BF, device=dev), 0, 7, 0.02, first=123)
# (cuBLAS writes its output with TMA stores, which initcheck does not count as initialisation: copy it
# through a plain kernel so the router's reads are not reported)
lg = torch.mm(h, wr.t(), out_dtype=torch.float32).mul(1.0)
ops.router_topk(None, None, ws, k, 0, logits_in=lg)
ops.permute(h, ws, xp)
hf = torch.zeros(T * k, f, dtype=BF, device=dev)
y = torch.zeros(T * k, d, dtype=BF, device=dev)
ops.moe_gemm_gate_up(wgu, xp, ws.offsets, hf)
ops.moe_gemm_down(wd, hf, ws.offsets, y)
sync = torch.zeros(257, dtype=torch.int32, device=dev)
ops.moe_ffn(wgu, wd, xp, ws.offsets, hf, y, sync)
out = torch.zeros(T, d, dtype=BF, device=dev)
ops.unpermute_combine(y, ws, out, T, residual=x, norm_w=ln, eps=1e-5, norm_out=torch.zeros_like(out))
# GQA decode attention + RoPE append
B, Hq, Hkv, hd, ctx = 3, 8, 2, 128, 70
page = ops.kv_page_size()
pps = math.ceil((ctx + 1) / page)
kc = torch.zeros(B * pps * Hkv * hd * page, dtype=BF, device=dev)
vc = torch.zeros_like(kc)
bt = torch.arange(B * pps, dtype=torch.int32, device=dev).view(B, pps)
pos = torch.full((B,), ctx, dtype=torch.int32, device=dev)
lens = torch.zeros(B + 4, dtype=torch.int32, device=dev)
qkv = uniform_bf16((B, (Hq + 2 * Hkv) * hd), 0, 6, 1.0).to(dev)
freqs = torch.outer(torch.arange(pps * page).float(), 1.0 / (10000 ** (torch.arange(0, hd, 2).float() / hd)))
cos_t, sin_t = freqs.cos().contiguous().to(dev), freqs.sin().contiguous().to(dev)
q = torch.zeros(B, Hq * hd, dtype=BF, device=dev)
ops.rope_append_gqa(qkv, 0, pos, cos_t, sin_t, Hq, Hkv, hd, bt, kc, vc, q, lens)
att = torch.zeros(B, Hq * hd, dtype=BF, device=dev)
ops.decode_attn_gqa(q, kc, vc, bt, lens[:B], Hq, Hkv, hd, att)
# MLA decode attention
H, R, RP = 16, 512, 64
mp = nat.value("mgb_mla_page_size")
mpps = math.ceil((ctx + 1) / mp)
cache = torch.zeros(B * mpps * nat.value("mgb_mla_page_elems", R, RP), dtype=BF, device=dev)
mbt = torch.arange(B * mpps, dtype=torch.int32, device=dev).view(B, mpps)
qm = uniform_bf16((B, H, 128 + RP), 0, 7, 1.0).to(dev)
ckv = uniform_bf16((B, R + RP), 0, 8, 1.0).to(dev)
nw = torch.ones(R, dtype=BF, device=dev)
fr = torch.outer(torch.arange(mpps * mp).float(), 1.0 / (10000 ** (torch.arange(0, RP, 2).float() / RP)))
mc, ms = fr.cos().contiguous().to(dev), fr.sin().contiguous().to(dev)
qn = torch.zeros(H, B, 128, dtype=BF, device=dev)
qpe = torch.zeros(B, H, RP, dtype=BF, device=dev)
mlens = torch.zeros(B + 4, dtype=torch.int32, device=dev)
nat.call("mgb_mla_append", qm.data_ptr(), ckv.data_ptr(), nw.data_ptr(), 1e-6, B, H, R, RP, 128, pos.data_ptr(),
         mc.data_ptr(), ms.data_ptr(), mbt.data_ptr(), mpps, cache.data_ptr(), qn.data_ptr(), qpe.data_ptr(),
         mlens.data_ptr(), st())
qlat = uniform_bf16((H, B, R), 0, 9, 0.5).to(dev)
olat = torch.zeros(H, B, R, dtype=BF, device=dev)
nat.call("mgb_decode_attn_mla", qlat.data_ptr(), qpe.data_ptr(), cache.data_ptr(), mbt.data_ptr(), mpps,
         mlens.data_ptr(), B, H, R, RP, 192 ** -0.5, olat.data_ptr(), st())
# prefill attention (GQA)
n_seq, P = 2, 130
qq = uniform_bf16((n_seq * P, Hq * hd), 0, 10, 1.0).to(dev)
kk = uniform_bf16((n_seq * P, Hkv * hd), 0, 11, 1.0).to(dev)
vv = uniform_bf16((n_seq * P, Hkv * hd), 0, 12, 1.0).to(dev)
po = torch.zeros(n_seq * P, Hq * hd, dtype=BF, device=dev)
ops.prefill_attn(qq, kk, vv, po, n_seq, P, Hq, Hkv, hd, hd, hd ** -0.5, hd, hd, hd)
torch.cuda.synchronize()
ops.capacity_status(reset=True)
print("sanitize smoke: all launches completed")
