"""Close the scheduler loop on a B200: measure the engine's module latency tables
(profiler.profile_engine), search the batching plan with them (plan_search.search, the reference's
search semantics), run the engine at the chosen plan and compare the measured forward time with the
plan's critical-path estimate (SURVEY.md §8c engine target 2).

  python tools/plan_b200.py --config mixtral-8x7b --kv-policy offload --out profiles/...json
"""
import argparse
import dataclasses
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_09716_b200.configs import get_arch  # noqa: E402
from paper_2503_09716_b200.engine import Engine  # noqa: E402
from paper_2503_09716_b200.plan_search import SearchSpace, evaluate_plan, search  # noqa: E402
from paper_2503_09716_b200.planner import (Hardware, ModelSpec, WorkloadSpec, footprint,  # noqa: E402
                                           load_profile_document)
from paper_2503_09716_b200.profiler import profile_engine  # noqa: E402
from paper_2503_09716_b200.schedule import latency_from_curves  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="mixtral-8x7b")
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--kv-policy", default="offload", choices=["offload", "resident"])
ap.add_argument("--host-gb", type=float, default=170.0)
ap.add_argument("--reserve-gb", type=float, default=12.0)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--profile-in", default=None)
ap.add_argument("--cpu-attention", action="store_true", help="profile the host-core attention and search omega")
ap.add_argument("--measured-memory", action="store_true",
                help="plan with the activation coefficients fitted to the profile's per-module memory tables")
ap.add_argument("--out", default=None)
args = ap.parse_args()

full = get_arch(args.config)
arch = full if args.layers is None else dataclasses.replace(full, layers=args.layers, name=f"{full.name}[{args.layers}L]")
t0 = time.time()
if args.profile_in:
    prof = json.load(open(args.profile_in))
else:
    prof = profile_engine(arch, token_grid=[2 ** i for i in range(0, 14)],
                          cpu_token_grid=[16, 64, 256, 1024] if args.cpu_attention else ())
    if args.out:
        with open(args.out + ".profile.json", "w") as f:
            json.dump(prof, f)
t_prof = time.time() - t0
hw, curves = load_profile_document(prof)
hw = Hardware(**{**hw.__dict__, "m_g": hw.m_g - int(args.reserve_gb * 2**30), "m_c": int(args.host_gb * 1e9)})
lat = latency_from_curves(curves)
spec_doc = arch.model_spec_document()
if args.measured_memory and "activation_coefficients" in prof:
    spec_doc = {**spec_doc, **prof["activation_coefficients"]}
spec = ModelSpec.from_document(spec_doc)
wl = WorkloadSpec(512, 256, 1_000_000, "decode")
omegas = tuple(round(0.1 * i, 1) for i in range(9)) if args.cpu_attention else (0.0,)
space = SearchSpace(b_a_grid=(64, 128, 256, 512, 1024), b_e_grid=(1024, 4096, 16384), omega_grid=omegas,
                    s_expert_slots_grid=(2, 4, 8), s_params_fracs=(0.0, 0.25, 0.5, 0.75, 1.0))
t0 = time.time()
best = search(spec, hw, lat, wl, space, kv_policy=args.kv_policy)
t_search = time.time() - t0
plan = best.plan
print("plan", plan, "predicted", best.t_forward, flush=True)
torch.cuda.synchronize()
mem0 = torch.cuda.memory_allocated()
torch.cuda.reset_peak_memory_stats()
eng = Engine(arch, plan, prompt_len=512, decode_len=256, use_graph=True, kv_policy=args.kv_policy)
eng.synthetic_prefill()
# the planner prices attention at the full context (max_context, offload_dag.py:353): time the last
# steps of the decode phase
eng.reset(768 - 2 - args.steps)
eng.buf.next_ids.random_(0, arch.vocab)
eng.capture()
eng.run_step()  # graph replay through the engine (primes the lookahead copies, checks the position)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(args.steps):
    eng.run_step()
e1.record()
torch.cuda.synchronize()
t_meas = e0.elapsed_time(e1) * 1e-3 / args.steps
# the GPU memory the run actually held (torch allocator peak, engine construction through the timed
# steps) next to the memory model's Eq. 3 total for the same plan
peak_gpu = torch.cuda.max_memory_allocated() - mem0
fp = footprint(spec, hw, wl, plan, kv_policy=args.kv_policy)
base = None
if args.cpu_attention:  # the best all-GPU plan of the same search, for the omega > 0 gain
    base = search(spec, hw, lat, wl, dataclasses.replace(space, omega_grid=(0.0,)), kv_policy=args.kv_policy)
out = {"config": arch.name, "kv_policy": args.kv_policy, "plan": plan.to_document(),
       "omega0_plan": base.plan.to_document() if base else None,
       "omega0_predicted_tokens_per_s": base.throughput if base else None,
       "predicted_forward_s": best.t_forward, "measured_forward_s": t_meas,
       "predicted_tokens_per_s": best.throughput, "measured_tokens_per_s": plan.B / t_meas,
       "rel_err": (t_meas - best.t_forward) / best.t_forward,
       "peak_gpu_bytes": peak_gpu, "model_gpu_bytes": fp.gpu_total, "model_s_is": fp.s_is,
       "activation_coefficients": prof.get("activation_coefficients"), "measured_memory": args.measured_memory,
       "profile_s": t_prof, "search_s": t_search, "hardware": prof["hardware"]}
print(json.dumps(out))
if args.out:
    with open(args.out, "w") as f:
        json.dump({"result": out, "profile": prof}, f)
