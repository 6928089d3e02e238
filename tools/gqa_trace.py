"""Per-page timeline of CTA 0 of the GQA decode kernel (variant build with -DMGB_GQA_TRACE):
  python tools/build_variant.py /tmp/gqa_tr.so -DMGB_GQA_TRACE
  MGB_LIB=/tmp/gqa_tr.so python tools/gqa_trace.py [B] [ctx]"""
import ctypes
import math
import os
import statistics
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
for _ in range(3):
    nat.call("mgb_decode_attn_gqa", q.data_ptr(), kc.data_ptr(), vc.data_ptr(), bt.data_ptr(), pps, lens.data_ptr(),
             B, HQ, HKV, HD, HD ** -0.5, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
lib = nat.LIB.load()
buf = (ctypes.c_ulonglong * (8 * 512))()
assert lib.mgb_gqa_trace_read(buf) == 0
ev = [[buf[e * 512 + i] for i in range(512)] for e in range(8)]
t0 = min(v for v in ev[0] if v)
n = sum(1 for v in ev[2] if v)
d = lambda a, b, rng: statistics.median((ev[b][i] - ev[a][i]) / 1e3 for i in rng if ev[a][i] and ev[b][i])  # noqa: E731
rng = range(20, max(21, n - 20))
print(f"pages {n}: load->landed(consumer) {d(0, 1, rng):.2f} us, landed->released {d(1, 2, rng):.2f} us, "
      f"page period {statistics.median((ev[1][i + 1] - ev[1][i]) / 1e3 for i in rng):.2f} us")
items = [i for i in range(512) if ev[5][i]]
print(f"items {len(items)}: merge {statistics.median((ev[6][i] - ev[5][i]) / 1e3 for i in items):.2f} us, "
      f"item period {statistics.median((ev[4][i + 1] - ev[4][i]) / 1e3 for i in items[:-1]):.2f} us, "
      f"kernel span {(max(v for v in ev[6] if v) - t0) / 1e3:.1f} us")
