"""Profiling driver: Mixtral-8x7B engine at the bench batch, synthetic prefill, N eager decode
forwards inside an NVTX range "decode_step" (for ncu --nvtx-include decode_step/)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_2503_09716_b200.configs import get_arch  # noqa: E402
from paper_2503_09716_b200.engine import Engine, resident_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral-8x7b")
ap.add_argument("--batch", type=int, default=None)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--reserve-gb", type=float, default=None, help="default: bench.py's measured per-model reserve")
args = ap.parse_args()
arch = get_arch(args.config)
import bench  # noqa: E402

plan = resident_plan(arch, 512, 256, B=args.batch, reserve_bytes=bench.reserve_bytes(args, arch))
eng = Engine(arch, plan, prompt_len=512, decode_len=256, use_graph=False)
eng.synthetic_prefill()
eng.reset(640)
eng.buf.next_ids.random_(0, arch.vocab)
torch.cuda.synchronize()
for i in range(args.steps):
    torch.cuda.nvtx.range_push("decode_step")
    eng.run_step()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
print("B", eng.B, "done")
