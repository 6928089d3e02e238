"""Golden results of the reference planner's batching-strategy search (plan_search.py:122-314),
generated from /root/reference itself in the build container:

  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_search.py

For each case: the model, hardware profile (synthesized tables), workload, search space, and the
reference's `search` winner (plan, t_forward, throughput), its candidate count and skip tallies
(`enumerate_candidates`), plus `model_based_baseline`.  tests/test_plan_search.py re-runs
paper_2503_09716_b200.plan_search on the same inputs and demands the same winners.
"""

from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import moe_planner as mp  # noqa: E402
from moe_planner.hw_profile import profile_to_document  # noqa: E402
from moe_planner.plan_search import SearchSpace, enumerate_candidates, model_based_baseline, search  # noqa: E402


def _plan(p):
    return {"B": p.B, "b_a": p.b_a, "b_e": p.b_e, "omega": p.omega, "s_expert": p.s_expert, "s_params": p.s_params}


def _space(s):
    return {"b_a_grid": list(s.b_a_grid), "b_e_grid": list(s.b_e_grid), "omega_grid": list(s.omega_grid),
            "s_expert_slots_grid": list(s.s_expert_slots_grid), "s_params_fracs": list(s.s_params_fracs),
            "prefill_B_grid": None if s.prefill_B_grid is None else list(s.prefill_B_grid)}


def main():
    from paper_2503_09716_b200.configs import DSV2_LITE, MIXTRAL_8X22B

    cases = []
    tiny, tiny_hw = mp.preset("tiny-test"), mp.tiny_test_hw()
    cases.append(("tiny_decode", tiny, tiny_hw, mp.WorkloadSpec(64, 32, 1024, "decode"), SearchSpace(), "decode"))
    cases.append(("tiny_prefill", tiny, tiny_hw, mp.WorkloadSpec(64, 32, 1024, "decode"),
                  SearchSpace(), "prefill"))
    mix = mp.preset("mixtral-8x7b")
    cases.append(("mixtral_a5000_decode", mix, mp.a5000_like(256_000_000_000), mp.WorkloadSpec(512, 256, 10_000),
                  SearchSpace(), "decode"))
    # this framework's own model documents on a B200-shaped machine with 1 TB of host RAM
    hw_b200 = mp.HardwareProfile(m_g=180_000_000_000, m_c=1_000_000_000_000, bw_htod=51e9, bw_dtoh=47e9,
                                 gpu_peak_flops=1.6e15, gpu_mem_bw=6.5e12, gpu_launch_overhead=5e-6,
                                 cpu_attn_flops=0.0)
    small = SearchSpace(b_a_grid=(64, 256, 1024), b_e_grid=(1024, 4096), omega_grid=(0.0,),
                        s_expert_slots_grid=(2, 4, 8), s_params_fracs=(0.0, 0.5, 1.0))
    for arch in (MIXTRAL_8X22B, DSV2_LITE):
        m = mp.load_model_spec(arch.model_spec_document())
        cases.append((f"{arch.name}_b200_decode", m, hw_b200, mp.WorkloadSpec(512, 256, 100_000), small, "decode"))
    for name, model, hw, wl, space, phase in cases:
        tables = mp.synth_profile(hw, model)
        skips: dict = {}
        n = sum(1 for _ in enumerate_candidates(model, hw, wl, space, phase, skip_counts=skips))
        t0 = time.time()
        best = search(model, hw, tables, wl, space, phase)
        dt = time.time() - t0
        base = model_based_baseline(model, hw, tables, wl, phase)
        doc = {"name": name, "model": model.to_document(), "profile": profile_to_document(hw, tables),
               "workload": {"prompt_len": wl.prompt_len, "decode_len": wl.decode_len,
                            "num_sequences": wl.num_sequences, "phase": wl.phase.value},
               "phase": phase, "space": _space(space), "candidates": n, "skips": skips,
               "best": {"plan": _plan(best.plan), "t_forward": best.t_forward, "throughput": best.throughput},
               "baseline": {"plan": _plan(base.plan), "t_forward": base.t_forward, "throughput": base.throughput},
               "reference_search_seconds": dt}
        with open(os.path.join(HERE, f"search_{name}.json"), "w") as f:
            json.dump(doc, f, sort_keys=True)
        print(name, n, _plan(best.plan), round(dt, 2), "s", flush=True)


if __name__ == "__main__":
    main()
