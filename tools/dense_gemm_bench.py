"""Plain projection GEMMs of the decode step (y = x W^T, bf16) at the bench shapes: cuBLAS
(torch.mm) against the repo's tcgen05 grouped GEMM run as one E = 1 segment (mgb_moe_gemm_down's
plain epilogue).  CUDA events, us per call and TFLOP/s.

python tools/dense_gemm_bench.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import ops  # noqa: E402

SHAPES = [("dsv2lite q_proj", 6058, 3072, 2048), ("dsv2lite o_proj", 6058, 2048, 2048),
          ("dsv2lite lm_head", 6058, 102400, 2048), ("mixtral qkv", 827, 6144, 4096),
          ("mixtral wo", 827, 4096, 4096), ("mixtral lm_head", 827, 32000, 4096)]


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


for name, T, N, K in SHAPES:
    x = torch.randn(T, K, device="cuda").bfloat16()
    w = (torch.randn(N, K, device="cuda") * 0.02).bfloat16()
    y1 = torch.empty(T, N, device="cuda", dtype=torch.bfloat16)
    y2 = torch.empty_like(y1)
    seg = torch.tensor([0, T], dtype=torch.int32, device="cuda")
    fl = 2.0 * T * N * K
    t1 = timed(lambda: torch.mm(x, w.t(), out=y1))
    row = {"shape": name, "T": T, "N": N, "K": K, "cublas_us": round(t1, 1), "cublas_tflops": round(fl / t1 / 1e6, 0)}
    try:
        t2 = timed(lambda: ops.moe_gemm_down(w[None], x, seg, y2))
        err = float(((y1.float() - y2.float()).abs().max() / y1.float().abs().max()))
        row.update(mgb_us=round(t2, 1), mgb_tflops=round(fl / t2 / 1e6, 0), rel_err=err)
    except Exception as e:  # noqa: BLE001
        row["mgb_error"] = str(e)[:120]
    print(json.dumps(row), flush=True)
