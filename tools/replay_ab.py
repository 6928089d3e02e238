"""Replayed decode forward time for same-box A/Bs of engine switches (environment variables): the
bench's engine at the bench batch, N warm-up replays (long enough to reach the power-capped clock the
bench runs at), then M timed replays with CUDA events; prints one JSON line.

MGB_SHARED_STREAM=0 python tools/replay_ab.py deepseek-v2-lite [warm] [timed]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200.configs import get_arch  # noqa: E402
from paper_2503_09716_b200.engine import Engine, resident_plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b"
warm = int(sys.argv[2]) if len(sys.argv) > 2 else 100
n = int(sys.argv[3]) if len(sys.argv) > 3 else 100
arch = get_arch(cfg)
reserve = (6.25 if cfg == "mixtral-8x7b" else 14.0) * (1 << 30)  # bench.py's measured reserves
plan = resident_plan(arch, 512, 256, reserve_bytes=int(reserve))
eng = Engine(arch, plan, prompt_len=512, decode_len=256, use_graph=True)
eng.synthetic_prefill()
eng.capture()
eng.reset(512)
for _ in range(warm):
    eng.run_step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    eng.run_step()
e1.record()
torch.cuda.synchronize()
env = {k: v for k, v in os.environ.items() if k.startswith("MGB_")}
print(json.dumps({"config": cfg, "B": eng.B, "env": env, "forward_ms": e0.elapsed_time(e1) / n,
                  "tokens_per_s": eng.B * n / (e0.elapsed_time(e1) * 1e-3)}))
