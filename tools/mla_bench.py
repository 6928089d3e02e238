"""Absorbed-MLA decode kernel alone at the DeepSeek-V2-Lite bench shape (CUDA events).

python tools/mla_bench.py [B] [ctx] [H]   -> us per launch, latent-cache GB/s, fraction of HBM peak

The byte count is the latent cache read ONCE per sequence (the algorithmic bytes: every head group
of a sequence attends over the same latent rows), whatever the kernel's head-group split re-reads.
MGB_MLA_CLUSTER=1 runs the head groups of a sequence as one multicast cluster instead of independent
CTAs sharing the pages through L2.
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import _native as nat  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 6058
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 540
H = int(sys.argv[3]) if len(sys.argv) > 3 else 16
RL, RP = 512, 64
page = nat.value("mgb_mla_page_size")
pps = math.ceil(CTX / page)
cache = torch.randn(B * pps * (RL + RP) * page, device="cuda").bfloat16()
bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
lens = torch.full((B,), CTX, dtype=torch.int32, device="cuda")
q_lat = torch.randn(H, B, RL, device="cuda").bfloat16()
q_pe = torch.randn(B, H, RP, device="cuda").bfloat16()
out = torch.empty(H, B, RL, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream


def run():
    nat.call("mgb_decode_attn_mla", q_lat.data_ptr(), q_pe.data_ptr(), cache.data_ptr(), bt.data_ptr(), pps,
             lens.data_ptr(), B, H, RL, RP, 192 ** -0.5, out.data_ptr(), st)


reps = int(os.environ.get("REPS", "20"))
for _ in range(3):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / reps * 1e3
byts = B * CTX * (RL + RP) * 2
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
hbm = next(v for k, v in peak.items() if "hbm" in k.lower() and isinstance(v, (int, float)))
print(f"B={B} ctx={CTX} H={H} page={page} cluster={os.environ.get('MGB_MLA_CLUSTER', '0')}: {us:.1f} us  "
      f"{byts / us / 1e3:.0f} GB/s  ({byts / us / 1e3 / hbm:.2f} of {hbm} GB/s)")
