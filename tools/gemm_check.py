"""Scratch GPU check of the tcgen05 grouped expert FFN (correctness + timing)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2503_09716_b200 import _native as nat  # noqa: E402


def ref_ffn(x, wgu, wd, offs):
    E = wgu.shape[0]
    f = wgu.shape[1] // 2
    H = torch.zeros(x.shape[0], f, dtype=torch.bfloat16, device=x.device)
    Y = torch.zeros(x.shape[0], wd.shape[1], dtype=torch.bfloat16, device=x.device)
    for e in range(E):
        a, b = offs[e], offs[e + 1]
        if b == a:
            continue
        xe = x[a:b].float()
        g = (xe @ wgu[e, :f].float().T).bfloat16().float()
        u = (xe @ wgu[e, f:].float().T).bfloat16().float()
        s = torch.nn.functional.silu(g).bfloat16().float()
        h = (s * u).bfloat16()
        H[a:b] = h
        Y[a:b] = (h.float() @ wd[e].float().T).bfloat16()
    return H, Y


def run(E, d, f, counts, check=True, iters=0):
    dev = "cuda"
    torch.manual_seed(0)
    offs = [0]
    for c in counts:
        offs.append(offs[-1] + c)
    rows = offs[-1]
    cap = rows + 256
    x = (torch.randn(cap, d, device=dev) * 0.5).bfloat16()
    wgu = (torch.randn(E, 2 * f, d, device=dev) * 0.02).bfloat16()
    wd = (torch.randn(E, d, f, device=dev) * 0.02).bfloat16()
    offs_t = torch.tensor(offs, dtype=torch.int32, device=dev)
    H = torch.zeros(cap, f, dtype=torch.bfloat16, device=dev)
    Y = torch.zeros(cap, d, dtype=torch.bfloat16, device=dev)
    s = torch.cuda.current_stream().cuda_stream
    nat.call("mgb_moe_gemm_gate_up", wgu.data_ptr(), x.data_ptr(), offs_t.data_ptr(), E, d, f, cap, H.data_ptr(), s)
    nat.call("mgb_moe_gemm_down", wd.data_ptr(), H.data_ptr(), offs_t.data_ptr(), E, d, f, cap, Y.data_ptr(), s)
    torch.cuda.synchronize()
    if check:
        Hr, Yr = ref_ffn(x[:rows], wgu, wd, offs)
        dh = (H[:rows].float() - Hr[:rows].float()).abs().max().item()
        dy = (Y[:rows].float() - Yr[:rows].float()).abs().max().item()
        sh = Hr.float().abs().max().item()
        sy = Yr.float().abs().max().item()
        print(f"E={E} d={d} f={f} counts={counts[:8]}.. maxdiff H {dh:.3e} (scale {sh:.3e}) Y {dy:.3e} (scale {sy:.3e})")
    if iters:
        ev0, ev1, ev2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        for _ in range(3):
            nat.call("mgb_moe_gemm_gate_up", wgu.data_ptr(), x.data_ptr(), offs_t.data_ptr(), E, d, f, cap, H.data_ptr(), s)
            nat.call("mgb_moe_gemm_down", wd.data_ptr(), H.data_ptr(), offs_t.data_ptr(), E, d, f, cap, Y.data_ptr(), s)
        t1 = t2 = 0.0
        for _ in range(iters):
            ev0.record()
            nat.call("mgb_moe_gemm_gate_up", wgu.data_ptr(), x.data_ptr(), offs_t.data_ptr(), E, d, f, cap, H.data_ptr(), s)
            ev1.record()
            nat.call("mgb_moe_gemm_down", wd.data_ptr(), H.data_ptr(), offs_t.data_ptr(), E, d, f, cap, Y.data_ptr(), s)
            ev2.record()
            torch.cuda.synchronize()
            t1 += ev0.elapsed_time(ev1)
            t2 += ev1.elapsed_time(ev2)
        t1 /= iters
        t2 /= iters
        t3 = 0.0
        for _ in range(iters):  # down alone, back to back (no gate/up in between)
            ev1.record()
            nat.call("mgb_moe_gemm_down", wd.data_ptr(), H.data_ptr(), offs_t.data_ptr(), E, d, f, cap, Y.data_ptr(), s)
            ev2.record()
            torch.cuda.synchronize()
            t3 += ev1.elapsed_time(ev2)
        t3 /= iters
        nz = sum(1 for c in counts if c > 0)
        b1 = nz * 2 * f * d * 2
        b2 = nz * d * f * 2
        fl1 = 2 * rows * d * 2 * f
        fl2 = 2 * rows * d * f
        print(f"  gate_up {t1*1e3:.1f} us  {b1/t1/1e6:.0f} GB/s  {fl1/t1/1e9:.0f} TF/s | down {t2*1e3:.1f} us {b2/t2/1e6:.0f} GB/s {fl2/t2/1e9:.0f} TF/s | down alone {t3*1e3:.1f} us")


SHAPES = {  # bench shapes: tokens per expert at the planner's batch
    "mixtral": (8, 4096, 14336, [208] * 8),
    "dsv2": (64, 2048, 1408, [568] * 64),
}

if __name__ == "__main__":
    if len(sys.argv) > 1:
        E, d, f, counts = SHAPES[sys.argv[1]]
        run(E, d, f, counts, check=len(sys.argv) > 2, iters=10)
        sys.exit(0)
    run(1, 256, 512, [40])
    run(8, 256, 512, [0, 1, 17, 33, 64, 100, 255, 300])
    run(4, 512, 384, [256, 257, 512, 3])
    run(8, 4096, 14336, [128, 120, 131, 140, 119, 125, 130, 131], iters=10)
    run(8, 4096, 14336, [190] * 8, iters=10)
    run(64, 2048, 1408, [48] * 64, iters=10)
    run(8, 4096, 14336, [1024] * 8, iters=5)
