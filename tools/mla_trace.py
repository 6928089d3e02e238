"""Per-page timeline of CTA 0 of the MLA decode kernel (build variant with -DMGB_MLA_TRACE):
  MGB_LIB=paper_2503_09716_b200/_lib/libmgb_trace.so python tools/mla_trace.py [B] [ctx]
Events per page: 0 load issued (stage free), 1 S issued (page landed), 2 P.V issued, 3 S ready at
softmax, 4 P written, 5 P.V done (O pulled)."""
import ctypes
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import _native as nat  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 6058
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 640
H, RL, RP = 16, 512, 64
page = nat.value("mgb_mla_page_size")
pps = math.ceil(CTX / page)
cache = torch.randn(B * pps * (RL + RP) * page, device="cuda").bfloat16()
bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
lens = torch.full((B,), CTX, dtype=torch.int32, device="cuda")
q_lat = torch.randn(H, B, RL, device="cuda").bfloat16()
q_pe = torch.randn(B, H, RP, device="cuda").bfloat16()
out = torch.empty(H, B, RL, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    nat.call("mgb_decode_attn_mla", q_lat.data_ptr(), q_pe.data_ptr(), cache.data_ptr(), bt.data_ptr(), pps,
             lens.data_ptr(), B, H, RL, RP, 192 ** -0.5, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
lib = nat.LIB.load()
buf = (ctypes.c_ulonglong * (16 * 256))()
assert lib.mgb_mla_trace_read(buf) == 0
N = 256
ev = [[buf[e * N + p] for p in range(N)] for e in range(15)]
t0 = min(v for v in ev[0] if v)
names = ["load", "S_iss", "PV_iss", "S_rdy", "P_wr", "PV_done"]
print("page " + " ".join(f"{n:>8}" for n in names) + "   (us from the first load; per-page deltas below)")
for p in range(40, 64):
    print(f"{p:4d} " + " ".join(f"{(ev[e][p] - t0) / 1e3:8.2f}" if ev[e][p] else "       -" for e in range(6)))
import statistics  # noqa: E402
def d(a, b, lo=20, hi=200):
    return statistics.median((ev[b][p] - ev[a][p]) / 1e3 for p in range(lo, hi) if ev[a][p] and ev[b][p])
print("median per page (us): load->S_iss %.2f  S_iss->S_rdy %.2f  S_rdy->P_wr %.2f  P_wr->PV_iss %.2f  PV_iss->PV_done %.2f" % (
    d(0, 1), d(1, 3), d(3, 4), d(4, 2), d(2, 5)))
print("P written by warp 4 (heads 8-15) after warp 0 (us): %.2f; later of the two -> PV_iss %.2f" % (
    d(4, 6), statistics.median((ev[2][p] - max(ev[4][p], ev[6][p])) / 1e3 for p in range(20, 200))))
print("page period (us): %.2f" % statistics.median((ev[0][p + 1] - ev[0][p]) / 1e3 for p in range(20, 200)))

ends = [p for p in range(N) if ev[9][p]]
for p in ends[2:8]:
    q = p + 1
    print(f"item end page {p}: last O pulled {(ev[9][p]-t0)/1e3:.2f}  stores issued +{(ev[10][p]-ev[9][p])/1e3:.2f}  "
          f"epilogue done +{(ev[11][p]-ev[9][p])/1e3:.2f}  next len loaded +{(ev[12][q]-ev[9][p])/1e3:.2f}  "
          f"next S ready +{(ev[3][q]-ev[9][p])/1e3:.2f}  (next S issued at {(ev[1][q]-ev[9][p])/1e3:+.2f}, "
          f"PV of last page issued {(ev[2][p]-ev[9][p])/1e3:+.2f})")
