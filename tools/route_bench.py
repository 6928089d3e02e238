"""Decode routing front end at the bench shapes (CUDA events, us per call): the fused mgb_moe_route
against the unfused chain add_rmsnorm + cuBLAS fp32 logits + router_topk + permute.

python tools/route_bench.py   -> one JSON line per shape
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200 import ops  # noqa: E402

BF16 = torch.bfloat16
SHAPES = [("mixtral-8x7b", 827, 4096, 8, 2, 0, 1, 1), ("mixtral-8x7b", 909, 4096, 8, 2, 0, 1, 1), ("deepseek-v2-lite", 6058, 2048, 64, 6, 1, 1, 1),
          ("mixtral-8x22b", 271, 6144, 8, 2, 0, 1, 1), ("deepseek-v2", 1024, 5120, 160, 6, 2, 8, 3)]


def timed(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


ONLY = sys.argv[1].split(",") if len(sys.argv) > 1 else None
for name, T, d, E, k, mode, ng, tg in SHAPES:
    if ONLY and name not in ONLY:
        continue
    x = torch.randn(T, d, device="cuda").to(BF16)
    o = torch.randn(T, d, device="cuda").to(BF16)
    ln = torch.ones(d, device="cuda", dtype=BF16)
    wr = (torch.randn(E, d, device="cuda") * 0.02).to(BF16)
    ws = ops.RouterWorkspace(T, E, k)
    h = torch.empty(T, d, device="cuda", dtype=BF16)
    xo = torch.empty_like(h)
    xp = torch.empty(T * k, d, device="cuda", dtype=BF16)
    lg = torch.empty(T, E, device="cuda", dtype=torch.float32)
    row = {"shape": name, "T": T, "d": d, "E": E, "k": k}
    if ops.moe_route_supported(T, d, E):
        row["fused_us"] = timed(lambda: ops.moe_route(x, o, ln, 1e-5, h, wr, ws, xp, mode, 1.0, ng, tg, x_out=xo,
                                                      logits_out=lg))
        # as the engine's decode step calls it: no h_out when one pass covers T, no logits copy
        h_eng = None if ops.moe_route_single_pass(T, d, E) else h
        row["engine_call_us"] = timed(lambda: ops.moe_route(x, o, ln, 1e-5, h_eng, wr, ws, xp, mode, 1.0, ng, tg,
                                                            x_out=xo))
        row["bulk_perm"] = os.environ.get("MGB_ROUTE_BULK", "0")

    def unfused():
        ops.add_rmsnorm(x, ln, 1e-5, h, delta=o, x_out=xo)
        torch.mm(h, wr.t(), out_dtype=torch.float32, out=lg)
        ops.router_topk(None, None, ws, k, mode, 1.0, ng, tg, logits_in=lg)
        ops.permute(h, ws, xp)
    if "fused_us" in row:  # per-phase split of one launch (globaltimer stamps, mgb_moe_route_stamps)
        from paper_2503_09716_b200 import _native as nat
        st = torch.zeros(1024, 16, dtype=torch.int64, device="cuda")
        nat.call("mgb_moe_route_stamps", st.data_ptr())
        ops.moe_route(x, o, ln, 1e-5, h_eng, wr, ws, xp, mode, 1.0, ng, tg, x_out=xo)
        torch.cuda.synchronize()
        nat.call("mgb_moe_route_stamps", None)
        st = st[(st[:, 9] > 0)].double()
        t0 = st[:, 9].min()
        names = {9: "start", 0: "lnw_staged", 1: "norm", 2: "logits", 3: "topk", 4: "hist", 5: "phase1_end",
                 6: "barrier_out", 7: "scan", 8: "end"}
        row["phases_us_mean_since_first_cta"] = {names[i]: round(float((st[:, i] - t0).mean()) / 1e3, 2)
                                                 for i in (9, 0, 1, 2, 3, 4, 5, 6, 7, 8)}
        row["phases_us_max"] = {names[i]: round(float((st[:, i] - t0).max()) / 1e3, 2) for i in (9, 5, 6, 8)}
    row["unfused_us"] = timed(unfused)
    row["norm_us"] = timed(lambda: ops.add_rmsnorm(x, ln, 1e-5, h, delta=o, x_out=xo))
    row["logits_us"] = timed(lambda: torch.mm(h, wr.t(), out_dtype=torch.float32, out=lg))
    row["topk_us"] = timed(lambda: ops.router_topk(None, None, ws, k, mode, 1.0, ng, tg, logits_in=lg))
    row["permute_us"] = timed(lambda: ops.permute(h, ws, xp))
    print(json.dumps({k_: (round(v, 2) if isinstance(v, float) else v) for k_, v in row.items()}), flush=True)
