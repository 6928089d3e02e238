"""Standalone times of the Mixtral decode-batch per-token kernels (RoPE/KV append, combine) at B=909:
MGB_ROPE_TPT / MGB_LIB A/Bs of their launch shapes.  python tools/smallk_bench.py"""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2503_09716_b200 import ops
from oracle.rng import uniform_bf16
BF16 = torch.bfloat16
def timed(fn, n=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
B, Hq, Hkv, hd = 909, 32, 8, 128
page = ops.kv_page_size(); pps = 12
qkv = uniform_bf16((B, (Hq + 2 * Hkv) * hd), 1, 2, 1.0).cuda()
fr = torch.arange(pps * page).float()[:, None] * (1.0 / (1e6 ** (torch.arange(0, hd, 2).float() / hd)))[None]
cos_t, sin_t = fr.cos().cuda(), fr.sin().cuda()
kc = torch.zeros(B * pps * Hkv * hd * page, dtype=BF16, device="cuda"); vc = torch.zeros_like(kc)
qo = torch.zeros(B, Hq * hd, dtype=BF16, device="cuda")
bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
pos = torch.full((B,), 640, dtype=torch.int32, device="cuda"); lens = torch.zeros(B, dtype=torch.int32, device="cuda")
r = {"env": {k: v for k, v in os.environ.items() if k.startswith("MGB_")}}
r["rope_us"] = timed(lambda: ops.rope_append_gqa(qkv, 0, pos, cos_t, sin_t, Hq, Hkv, hd, bt, kc, vc, qo, lens))
d, k, E = 4096, 2, 8
ws = ops.RouterWorkspace(B, E, k)
x = uniform_bf16((B, d), 3, 4, 1.0).cuda(); o = uniform_bf16((B, d), 3, 5, 1.0).cuda()
ln = torch.ones(d, dtype=BF16, device="cuda"); wr = uniform_bf16((E, d), 3, 6, 0.05).cuda()
xp = torch.empty(B * k, d, dtype=BF16, device="cuda")
ops.moe_route(x, o, ln, 1e-5, None if ops.moe_route_single_pass(B, d, E) else torch.empty_like(x), wr, ws, xp, 0, x_out=torch.empty_like(x))
yp = uniform_bf16((B * k, d), 3, 7, 1.0).cuda(); xo = x.clone(); h = torch.empty_like(x)
r["combine_us"] = timed(lambda: ops.unpermute_combine(yp, ws, xo, B, residual=x, norm_w=ln, eps=1e-5, norm_out=h))
print(json.dumps(r))
