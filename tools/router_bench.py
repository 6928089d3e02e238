"""Router kernel timing vs T/E (CUDA events, 20 reps)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2503_09716_b200 import ops

def t(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

for T, d, E, k, mode in [(827, 4096, 8, 2, 0), (6058, 2048, 64, 6, 1), (1024, 5120, 160, 6, 2)]:
    x = torch.randn(T, d, device="cuda").bfloat16(); wg = (torch.randn(E, d, device="cuda") * 0.02).bfloat16()
    ws = ops.RouterWorkspace(T, E, k)
    lg = torch.mm(x, wg.t(), out_dtype=torch.float32)
    us_fused = t(lambda: ops.router_topk(x, wg, ws, k, mode, 1.0, 8, 3))
    us_lin = t(lambda: ops.router_topk(None, None, ws, k, mode, 1.0, 8, 3, logits_in=lg))
    us_mm = t(lambda: torch.mm(x, wg.t(), out_dtype=torch.float32))
    xp = torch.empty(T * k, d, device="cuda", dtype=torch.bfloat16)
    us_perm = t(lambda: ops.permute(x, ws, xp))
    print(f"T={T} d={d} E={E}: fused GEMV router {us_fused:.1f} us | logits_in router {us_lin:.1f} us | cuBLAS fp32-out gate GEMM {us_mm:.1f} us | permute {us_perm:.1f} us")
