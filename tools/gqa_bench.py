"""Paged GQA decode attention kernel alone at the Mixtral-8x7B bench shape (CUDA events).

python tools/gqa_bench.py [B] [ctx]   -> us per launch, KV GB/s, fraction of HBM peak
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import _native as nat  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 827
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 640
HQ, HKV, HD = 32, 8, 128
page = nat.value("mgb_kv_page_size")
pps = math.ceil(CTX / page)
kc = torch.randn(B * pps * HKV * HD * page, device="cuda").bfloat16()
vc = torch.randn_like(kc)
bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
lens = torch.full((B,), CTX, dtype=torch.int32, device="cuda")
q = torch.randn(B, HQ, HD, device="cuda").bfloat16()
out = torch.empty(B, HQ * HD, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream


def run():
    nat.call("mgb_decode_attn_gqa", q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(), pps, lens.data_ptr(),
             B, HQ, HKV, HD, HD ** -0.5, out.data_ptr(), st)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 20
e0.record()
for _ in range(n):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / n * 1e3
nbytes = B * CTX * HKV * HD * 2 * 2
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = next((v for k, v in peak.items() if "hbm" in k.lower() and isinstance(v, (int, float))), 6557.4)
print(f"B={B} ctx={CTX} page={page}: {us:.1f} us  {nbytes / us / 1e3:.0f} GB/s  ({nbytes / us / 1e3 / hbm:.2f} of {hbm} GB/s)")
