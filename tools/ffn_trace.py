"""Where the fused FFN kernel's roles wait (variant build with -DMGB_GEMM_TRACE):
  python tools/build_variant.py /tmp/ffn_tr.so -DMGB_GEMM_TRACE
  MGB_LIB=/tmp/ffn_tr.so python tools/ffn_trace.py [tokens_per_expert]
Per CTA: cycles in producer empty waits, MMA full waits (data not landed), MMA TMEM-empty waits
(epilogue behind), epilogue TMEM-full waits, producer dependency waits, and the kernel's cycles."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import _native as nat  # noqa: E402
from paper_2503_09716_b200 import ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 207
cfg = sys.argv[2] if len(sys.argv) > 2 else "mixtral-8x7b"  # deepseek-v2-lite: the two grouped launches
from paper_2503_09716_b200.configs import get_arch  # noqa: E402

_a = get_arch(cfg)
E, d, f = _a.n_experts, _a.hidden, _a.moe_ffn
fused = E <= 16
bf = torch.bfloat16
wgu = (torch.randn(E, 2 * f, d, device="cuda") * 0.02).to(bf)
wd = (torch.randn(E, d, f, device="cuda") * 0.02).to(bf)
T = n * E
x = torch.randn(T, d, device="cuda").to(bf)
h = torch.empty(T, f, device="cuda", dtype=bf)
y = torch.empty(T, d, device="cuda", dtype=bf)
offs = torch.arange(0, T + 1, n, dtype=torch.int32, device="cuda")
sync = torch.zeros(257, dtype=torch.int32, device="cuda")
lib = nat.LIB.load()
buf = (ctypes.c_longlong * (256 * 8))()
def run(which):
    if fused:
        ops.moe_ffn(wgu, wd, x, offs, h, y, sync)
    elif which == "gate_up":
        ops.moe_gemm_gate_up(wgu, x, offs, h)
    else:
        ops.moe_gemm_down(wd, h, offs, y)


which = sys.argv[3] if len(sys.argv) > 3 else "gate_up"
for _ in range(3):
    run(which)
torch.cuda.synchronize()
lib.mgb_ffn_trace_read(buf)
run(which)
torch.cuda.synchronize()
assert lib.mgb_ffn_trace_read(buf) == 0
rows = [[buf[c * 8 + i] for i in range(8)] for c in range(148)]
names = ["producer empty", "MMA full (data)", "MMA tmem-empty", "epilogue tmem-full", "producer dependency"]
lead = rows[0::2]
kc = sum(r[5] for r in rows) / len(rows)
print(f"kernel {kc:.0f} cycles per CTA (avg)")
for i, nm in enumerate(names):
    vals = [r[i] for r in (lead if i in (1, 2) else rows)]
    print(f"  {nm:22s}: {sum(vals) / len(vals) / kc:6.1%} of the kernel (avg over {'leader' if i in (1, 2) else 'all'} CTAs)")
