"""The grouped expert GEMMs at prefill-sized groups (module-based batching's b_e = 1,024-8,192 tokens
per expert): Mixtral-8x7B / DeepSeek-V2-Lite expert dims, CUDA-event timed;
TFLOP/s and the fraction of the measured dense bf16 peak (MEASURED_PEAKS.json, burst).

python tools/gemm_prefill_bench.py [config] [tokens_per_expert,...] [ffn]   -> one JSON line per size
("ffn" also times the fused single-launch FFN, mgb_moe_ffn, on the same rows)
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_09716_b200 import ops  # noqa: E402
from paper_2503_09716_b200.configs import get_arch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b"
sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1024,2048,4096,8192").split(",")]
a = get_arch(cfg)
E, d, f = a.n_experts, a.hidden, a.moe_ffn
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
bf = torch.bfloat16
wgu = (torch.randn(E, 2 * f, d, device="cuda") * 0.02).to(bf)
wd = (torch.randn(E, d, f, device="cuda") * 0.02).to(bf)
reps = int(os.environ.get("REPS", "10"))
with_ffn = len(sys.argv) > 3 and sys.argv[3] == "ffn"
sync = torch.zeros(257, dtype=torch.int32, device="cuda")
for n in sizes:
    T = n * E
    x = torch.randn(T, d, device="cuda").to(bf)
    h = torch.empty(T, f, device="cuda", dtype=bf)
    y = torch.empty(T, d, device="cuda", dtype=bf)
    offs = torch.arange(0, T + 1, n, dtype=torch.int32, device="cuda")
    row = {"config": cfg, "tokens_per_expert": n, "E": E, "d": d, "f": f}
    cases = [("gate_up", lambda: ops.moe_gemm_gate_up(wgu, x, offs, h), 2.0 * T * d * 2 * f),
             ("down", lambda: ops.moe_gemm_down(wd, h, offs, y), 2.0 * T * f * d)]
    if with_ffn:
        cases.append(("ffn", lambda: ops.moe_ffn(wgu, wd, x, offs, h, y, sync), 2.0 * T * d * 3 * f))
    for name, fn, flops in cases:
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        tf = flops / (ms * 1e-3) / 1e12
        byts = E * 3 * f * d * 2 + T * (2 * d + 2 * f) * 2  # weights once + rows in/out of both GEMMs
        row[name] = {"ms": round(ms, 4), "tflops": round(tf, 1), "frac_of_bf16_peak": round(tf / peak, 3),
                     "ffn_gbs_if_all_weights": round(byts / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps(row), flush=True)
