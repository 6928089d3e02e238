"""Host-core throughput of the CPU attention (ATTN_MECH_CPU) at Mixtral shapes: KV GB/s read."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_09716_b200 import _native as nat  # noqa: E402

B, Hq, Hkv, hd, P = int(sys.argv[1]) if len(sys.argv) > 1 else 64, 32, 8, 128, 64
L, pps = 640, 12
kp = torch.randn(B * pps * Hkv * hd * P).to(torch.bfloat16)
vp = torch.randn(B * pps * Hkv * hd * P).to(torch.bfloat16)
q = torch.randn(B, Hq, hd).to(torch.bfloat16)
sl = torch.full((B,), L, dtype=torch.int32)
out = torch.zeros(B, Hq * hd, dtype=torch.bfloat16)
d = nat.CpuAttnGqa(kp.data_ptr(), vp.data_ptr(), q.data_ptr(), sl.data_ptr(), out.data_ptr(), 0, pps, B, Hq, Hkv, hd,
                   P, 0.088, 0)
nat.call("mgb_cpu_attn_gqa", ctypes.byref(d))
t = time.time()
n = 5
for _ in range(n):
    nat.call("mgb_cpu_attn_gqa", ctypes.byref(d))
dt = (time.time() - t) / n
by = B * L * Hkv * hd * 2 * 2
print(f"threads {nat.value('mgb_cpu_threads', 0)} simd {nat.value('mgb_cpu_attn_simd')} B={B}: {dt * 1e3:.2f} ms, "
      f"{by / dt / 1e9:.1f} GB/s of KV")
