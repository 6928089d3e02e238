"""Device memory of the bench configuration, phase by phase: what the engine holds beyond its
weights and paged KV (the planner's `reserve`), measured with the torch allocator stats and
cudaMemGetInfo (CUDA context, cuBLAS workspaces and graph pools included).

python tools/mem_probe.py [config] [reserve_gb] [batch]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200.configs import get_arch  # noqa: E402
from paper_2503_09716_b200.engine import Engine, resident_plan  # noqa: E402
from paper_2503_09716_b200.planner import ModelSpec  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "mixtral-8x7b"
reserve = float(sys.argv[2]) if len(sys.argv) > 2 else 14.0
batch = int(sys.argv[3]) if len(sys.argv) > 3 else None
arch = get_arch(cfg)
spec = ModelSpec.from_document(arch.model_spec_document())
P, N = 512, 256
free0, total = torch.cuda.mem_get_info()
plan = resident_plan(arch, P, N, B=batch, reserve_bytes=int(reserve * 2**30))
GB = 1e9
res = {"config": cfg, "reserve_gb": reserve, "B": plan.B, "hbm_total_gb": total / GB,
       "used_before_engine_gb": (total - free0) / GB,
       "weights_gb": spec.model_bytes / GB,
       "kv_gb": plan.B * (P + N) * spec.kv_bytes_per_token_layer * spec.num_layers / GB}


def snap(tag):
    torch.cuda.synchronize()
    free, _ = torch.cuda.mem_get_info()
    res[tag] = {"used_gb": round((total - free) / GB, 3), "alloc_gb": round(torch.cuda.memory_allocated() / GB, 3),
                "peak_alloc_gb": round(torch.cuda.max_memory_allocated() / GB, 3),
                "reserved_gb": round(torch.cuda.memory_reserved() / GB, 3)}


eng = Engine(arch, plan, prompt_len=P, decode_len=N, seed=0, use_graph=True)
snap("engine")
eng.synthetic_prefill(seed=1)
eng.capture()
snap("captured")
eng.reset(P)
for _ in range(4):
    eng.run_step()
snap("decode")
ids = torch.randint(0, arch.vocab, (plan.B, P), generator=torch.Generator().manual_seed(11))
eng.prefill(ids)
snap("prefill")
res["overhead_gb"] = res["prefill"]["used_gb"] - res["weights_gb"] - res["kv_gb"]
res["free_after_gb"] = torch.cuda.mem_get_info()[0] / GB
print(json.dumps(res))
