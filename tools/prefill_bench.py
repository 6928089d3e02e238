"""Batched prefill throughput (Engine.prefill) at the Mixtral-8x7B bench config: B sequences x P
prompt tokens through the prefill phase, CUDA-event timed; prompt tokens/s."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200.configs import get_arch  # noqa: E402
from paper_2503_09716_b200.engine import Engine, resident_plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral-8x7b")
ap.add_argument("--prompt-len", type=int, default=512)
ap.add_argument("--chunk-tokens", type=int, default=None, help="default: the engine's choice")
ap.add_argument("--reserve-gb", type=int, default=14)
args = ap.parse_args()
arch = get_arch(args.config)
plan = resident_plan(arch, args.prompt_len, 256, reserve_bytes=args.reserve_gb << 30)
eng = Engine(arch, plan, prompt_len=args.prompt_len, decode_len=256, use_graph=True)
ids = torch.randint(0, arch.vocab, (eng.B, args.prompt_len), generator=torch.Generator().manual_seed(0))
eng.prefill(ids, chunk_tokens=args.chunk_tokens)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
eng.prefill(ids, chunk_tokens=args.chunk_tokens)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e-3
print(json.dumps({"config": args.config, "B": eng.B, "prompt_len": args.prompt_len, "chunk_tokens": args.chunk_tokens,
                  "prefill_s": t, "prompt_tokens_per_s": eng.B * args.prompt_len / t}))
