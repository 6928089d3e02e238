"""Where the graph-replayed decode forward spends time beyond its kernels: one forward timed (a) as
a CUDA-graph replay, (b) issued eagerly behind a parked stream (host pre-enqueued), both with CUDA
events around the whole forward, at the bench batch and mid-decode context.

python tools/graph_gap.py [config]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200.configs import get_arch  # noqa: E402
from paper_2503_09716_b200.engine import Engine, resident_plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b"
arch = get_arch(cfg)
plan = resident_plan(arch, 512, 256, reserve_bytes=14 << 30)
eng = Engine(arch, plan, prompt_len=512, decode_len=256, use_graph=True)
eng.synthetic_prefill()
eng.capture()


def ev():
    return torch.cuda.Event(enable_timing=True)


res = {"config": cfg, "B": eng.B}
# graph replays
eng.reset(640)
for _ in range(3):
    eng.run_step()
torch.cuda.synchronize()
e0, e1 = ev(), ev()
n = 10
e0.record()
for _ in range(n):
    eng.run_step()
e1.record()
torch.cuda.synchronize()
res["graph_ms"] = e0.elapsed_time(e1) / n
# eager, host pre-enqueued behind a parked stream
st = eng.stream
ts = []
for _ in range(3):
    eng.reset(640)
    a, b = ev(), ev()
    with torch.cuda.stream(st):
        torch.cuda._sleep(int(3e8))
        a.record(st)
        eng._step(record=False)
        b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
res["eager_preenqueued_ms"] = min(ts)
print(json.dumps(res))

# per-launch times INSIDE a captured graph: external timing events around every libmgb / cuBLAS call
if len(sys.argv) > 2 and sys.argv[2] == "nodes":
    from paper_2503_09716_b200 import _native as nat

    pend = []

    def timed(name, fn):
        def inner(*a, **k):
            e0 = torch.cuda.Event(enable_timing=True, external=True)
            e1 = torch.cuda.Event(enable_timing=True, external=True)
            e0.record()
            r = fn(*a, **k)
            e1.record()
            pend.append((name if isinstance(name, str) else name(a), e0, e1))
            return r
        return inner

    orig, mm, bmm = nat.call, torch.mm, torch.bmm
    nat.call = timed(lambda a: a[0].replace("mgb_", ""), orig)
    torch.mm = timed("cublas_gemm", mm)
    torch.bmm = timed("cublas_bmm", bmm)
    eng.reset(640)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=eng.stream):
        eng._step(record=False)
    nat.call, torch.mm, torch.bmm = orig, mm, bmm
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    agg, gaps = {}, 0.0
    for i, (nm, e0, e1) in enumerate(pend):
        agg[nm] = agg.get(nm, 0.0) + e0.elapsed_time(e1)
        if i + 1 < len(pend):
            gaps += e1.elapsed_time(pend[i + 1][1])
    tot = pend[0][1].elapsed_time(pend[-1][2])
    print(json.dumps({"graph_with_events_ms": tot, "sum_nodes_ms": sum(agg.values()), "gaps_ms": gaps,
                      "per_kernel_ms": {k: round(v, 3) for k, v in sorted(agg.items(), key=lambda x: -x[1])}}))
