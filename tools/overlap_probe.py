"""Can the next attention micro-batch's QKV projection (cuBLAS, tensor-bound) hide under this
micro-batch's decode attention (HBM-bound)?  GQA attention over half the Mixtral bench batch on one
stream, the other half's QKV GEMM on a second stream, timed serial vs concurrent with CUDA events.
MGB_ATTN_SMS caps the SMs the attention grid spans, leaving the rest to the GEMM.

MGB_ATTN_SMS=120 python tools/overlap_probe.py [B_mb] [ctx]
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import ops  # noqa: E402
from paper_2503_09716_b200 import _native as nat  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 414
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 640
HQ, HKV, HD, D = 32, 8, 128, 4096
page = nat.value("mgb_kv_page_size")
pps = math.ceil(CTX / page)
kc = torch.randn(B * pps * HKV * HD * page, device="cuda").bfloat16()
vc = torch.randn_like(kc)
bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
lens = torch.full((B,), CTX, dtype=torch.int32, device="cuda")
q = torch.randn(B, HQ, HD, device="cuda").bfloat16()
out = torch.empty(B, HQ * HD, device="cuda", dtype=torch.bfloat16)
sched = torch.zeros(2, dtype=torch.int32, device="cuda")
x = torch.randn(B, D, device="cuda").bfloat16()
wqkv = (0.02 * torch.randn((HQ + 2 * HKV) * HD, D, device="cuda")).bfloat16()
qkv = torch.empty(B, wqkv.shape[0], device="cuda", dtype=torch.bfloat16)
s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()


def attn():
    ops.decode_attn_gqa(q, kc, vc, bt, lens, HQ, HKV, HD, out, sched=sched)


def gemm():
    torch.mm(x, wqkv.t(), out=qkv)


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def serial():
    attn()
    gemm()


fork, j0, j1 = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()


def concurrent():
    cur = torch.cuda.current_stream()
    fork.record(cur)
    s0.wait_event(fork)
    s1.wait_event(fork)
    with torch.cuda.stream(s0):
        attn()
    with torch.cuda.stream(s1):
        gemm()
    j0.record(s0)
    j1.record(s1)
    cur.wait_event(j0)
    cur.wait_event(j1)


res = {"B": B, "ctx": CTX, "attn_sms": os.environ.get("MGB_ATTN_SMS", "all"),
       "attn_us": timed(attn), "gemm_us": timed(gemm), "serial_us": timed(serial), "concurrent_us": timed(concurrent)}
res["saved_us"] = res["serial_us"] - res["concurrent_us"]
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}))
