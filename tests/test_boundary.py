"""The engine <-> reference planner boundary, both directions, on documents the reference itself
wrote or read (tests/golden/make_golden_sim.py):

  - profile out: the engine's MEASURED B200 profile documents (profiler.profile_engine, committed in
    profiles/r1_plan_*.json) are accepted by the reference's `ingest_profile`
    (hw_profile.py:156-216), and the reference's `evaluate_plan` on them gives the t_forward /
    throughput / feasibility this framework's planner computes from the same documents;
  - plan in: `plan.json` as written by the reference's `plan_to_doc` / `evaluation_to_doc`
    (cli.py:74-109) loads into this framework's BatchingPlan unchanged (the engine's plan input).
"""

import json
import math
import os

import pytest

from paper_2503_09716_b200.plan_search import evaluate_plan
from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec, WorkloadSpec, load_plan, load_profile_document
from paper_2503_09716_b200.schedule import latency_from_curves

HERE = os.path.join(os.path.dirname(__file__), "golden")
DOC = json.load(open(os.path.join(HERE, "boundary.json")))


@pytest.mark.parametrize("i", range(len(DOC["rows"])))
def test_measured_profile_evaluates_like_the_reference(i):
    row = DOC["rows"][i]
    spec = ModelSpec.from_document(row["model"])
    hw, curves = load_profile_document(DOC["profiles"][row["profile"]])
    w = row["workload"]
    wl = WorkloadSpec(w["prompt_len"], w["decode_len"], w["num_sequences"], row["phase"])
    ev = evaluate_plan(spec, hw, latency_from_curves(curves), wl, BatchingPlan.from_document(row["plan"]))
    ref = row["evaluation"]
    assert ev.feasible == ref["feasible"]
    if ref["t_forward"] is None:
        assert not math.isfinite(ev.t_forward)
    else:
        assert math.isclose(ev.t_forward, ref["t_forward"], rel_tol=1e-12)
        assert math.isclose(ev.throughput, ref["throughput"], rel_tol=1e-12)
    fp = ref["footprint"]
    assert (ev.footprint.s_kv_cpu, ev.footprint.s_kv_gpu, ev.footprint.gpu_total, ev.footprint.host_total) == \
        (fp["s_kv_cpu"], fp["s_kv_gpu"], fp["gpu_total"], fp["host_total"])


def test_profiles_are_monotone_reference_tables():
    """What ingest_profile additionally enforces (hw_profile.py:117-142): >= 2 token points per
    context, latency non-decreasing in tokens."""
    for name, prof in DOC["profiles"].items():
        for t in prof["latency_tables"]:
            by_ctx = {}
            for tok, ctx, lat in t["entries"]:
                by_ctx.setdefault(ctx, []).append((tok, lat))
            for ctx, pts in by_ctx.items():
                pts.sort()
                assert len(pts) >= 2, (name, t["module_kind"], ctx)
                assert all(b[1] >= a[1] for a, b in zip(pts, pts[1:])), (name, t["module_kind"], ctx)


@pytest.mark.parametrize("fname", ["plan_tiny_ref.json", "plan_tiny_ref_eval.json"])
def test_reference_written_plan_documents_load(fname):
    path = os.path.join(HERE, fname)
    plan = load_plan(path)
    assert plan == BatchingPlan(64, 32, 16, 0.0, 0, plan.s_params)
    from paper_2503_09716_b200.configs import TINY
    assert plan.s_params == ModelSpec.from_document(TINY.model_spec_document()).model_bytes
    with pytest.raises(ValueError):
        load_plan({"plan": {"B": 1}})
