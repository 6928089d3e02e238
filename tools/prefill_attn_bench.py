"""mgb_prefill_attn (tcgen05 causal prefill attention) vs torch SDPA on the prefill chunk shapes
of the bench configs: Mixtral-8x7B (64 prompts x 512, 32 q / 8 kv heads, hd 128) and
DeepSeek-V2-Lite (64 x 512, 16 heads, qk 192 = 128 nope + 64 shared rope, v 128).  CUDA-event
timed, causal FLOPs = 2 * n * H * P * (P + 1) / 2 * (d_qk + d_v)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import ops  # noqa: E402

BF16 = torch.bfloat16


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


rows = []
n, P = 64, 512
# GQA
Hq, Hkv, hd = 32, 8, 128
T = n * P
q = torch.randn(T, Hq * hd, device="cuda").to(BF16)
k = torch.randn(T, Hkv * hd, device="cuda").to(BF16)
v = torch.randn(T, Hkv * hd, device="cuda").to(BF16)
o = torch.empty(T, Hq * hd, device="cuda", dtype=BF16)
fl = 2 * n * Hq * P * (P + 1) / 2 * (hd + hd)
t_m = timed(lambda: ops.prefill_attn(q, k, v, o, n, P, Hq, Hkv, hd, hd, hd ** -0.5, hd, hd, hd))
t_s = timed(lambda: torch.nn.functional.scaled_dot_product_attention(
    q.view(n, P, Hq, hd).transpose(1, 2), k.view(n, P, Hkv, hd).transpose(1, 2), v.view(n, P, Hkv, hd).transpose(1, 2),
    is_causal=True, enable_gqa=True))
rows.append({"shape": "mixtral gqa 64x512 32/8 hd128", "mgb_ms": t_m * 1e3, "sdpa_ms": t_s * 1e3,
             "mgb_tflops": fl / t_m / 1e12, "sdpa_tflops": fl / t_s / 1e12})
# MLA
H, nope, r, vd = 16, 128, 64, 128
q = torch.randn(T, H * (nope + r), device="cuda").to(BF16)
kv = torch.randn(T, H * (nope + vd), device="cuda").to(BF16)
kpe = torch.randn(T, r, device="cuda").to(BF16)
o = torch.empty(T, H * vd, device="cuda", dtype=BF16)
kfull = torch.cat([kv.view(T, H, nope + vd)[..., :nope], kpe[:, None].expand(T, H, r)], -1).contiguous()
vv = kv.view(T, H, nope + vd)[..., nope:]
fl = 2 * n * H * P * (P + 1) / 2 * (nope + r + vd)
t_m = timed(lambda: ops.prefill_attn(q, kv, kv, o, n, P, H, H, nope + r, vd, (nope + r) ** -0.5, nope + r, nope + vd,
                                     nope + vd, v_col0=nope, kr=kpe))
t_s = timed(lambda: torch.nn.functional.scaled_dot_product_attention(
    q.view(n, P, H, nope + r).transpose(1, 2), kfull.view(n, P, H, nope + r).transpose(1, 2),
    vv.reshape(n, P, H, vd).transpose(1, 2), is_causal=True, scale=(nope + r) ** -0.5))
rows.append({"shape": "dsv2 mla 64x512 16 heads qk192 v128", "mgb_ms": t_m * 1e3, "sdpa_ms": t_s * 1e3,
             "mgb_tflops": fl / t_m / 1e12, "sdpa_tflops": fl / t_s / 1e12})
print(json.dumps(rows, indent=1))
