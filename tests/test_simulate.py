"""paper_2503_09716_b200.simulate vs the reference's own simulator (exec_sim.py:161-360) on
tests/golden/sim_*.json (tests/golden/make_golden_sim.py): the same report -- makespan, per-resource
busy / idle, link bytes, peak GPU occupancy, oom flag, per-expert token counts -- the same JSONL
trace, and the same simulator-vs-estimate gap, including on this engine's measured B200 profiles."""

import glob
import io
import json
import math
import os

import pytest

from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec, WorkloadSpec, load_profile_document
from paper_2503_09716_b200.schedule import latency_from_curves
from paper_2503_09716_b200.simulate import RoutingModel, compare_with_estimate, sample_routing, simulate_plan

HERE = os.path.join(os.path.dirname(__file__), "golden")
SIMS = sorted(glob.glob(os.path.join(HERE, "sim_*.json")))


def _close(a, b, tol=1e-12):
    return math.isclose(a, b, rel_tol=tol, abs_tol=1e-15)


@pytest.mark.parametrize("path", SIMS, ids=[os.path.basename(p) for p in SIMS])
def test_simulate_plan_matches_reference(path):
    doc = json.load(open(path))
    spec = ModelSpec.from_document(doc["model"])
    hw, curves = load_profile_document(doc["profile"])
    w = doc["workload"]
    wl = WorkloadSpec(w["prompt_len"], w["decode_len"], w["num_sequences"], w["phase"])
    plan = BatchingPlan.from_document(doc["plan"])
    r = doc["routing"]
    routing = RoutingModel(r["mode"], r["concentration"], r["seed"])
    buf = io.StringIO()
    rep = simulate_plan(spec, hw, latency_from_curves(curves), wl, plan, routing, trace_stream=buf).to_document()
    ref = doc["report"]
    assert rep["expert_tokens"] == ref["expert_tokens"]
    for k in ("makespan", "bytes_htod", "bytes_dtoh", "peak_gpu_bytes", "mean_tokens_per_expert", "throughput"):
        assert _close(rep[k], ref[k]), (k, rep[k], ref[k])
    for k in ("busy", "idle_fraction"):
        assert set(rep[k]) == set(ref[k])
        for res in ref[k]:
            assert _close(rep[k][res], ref[k][res]), (k, res)
    assert rep["oom_flag"] == ref["oom_flag"]
    if doc["trace"] is not None:
        mine = [json.loads(x) for x in buf.getvalue().splitlines()]
        theirs = [json.loads(x) for x in doc["trace"]]
        assert len(mine) == len(theirs)
        for a, b in zip(mine, theirs):
            assert (a["node"], a["kind"], a["resource"], a["action"]) == (b["node"], b["kind"], b["resource"], b["action"])
            assert _close(a["time"], b["time"])
    gap = compare_with_estimate(spec, hw, latency_from_curves(curves), wl, plan)
    assert gap <= 1e-3 and abs(gap - doc["compare_with_estimate"]) <= 1e-12


def test_sample_routing_even_and_sampled():
    doc = json.load(open(os.path.join(HERE, "sim_tiny_sampled.json")))
    spec = ModelSpec.from_document(doc["model"])
    rows = doc["report"]["expert_tokens"]
    r = doc["routing"]
    B = doc["plan"]["B"]
    for l, row in enumerate(rows):
        assert sample_routing(spec, B, RoutingModel(r["mode"], r["concentration"], r["seed"]), l) == row
        assert sum(row) == B * spec.top_k
    assert sample_routing(spec, 8, RoutingModel(), 0) == [8 * spec.top_k // spec.experts_per_layer] * spec.experts_per_layer
    with pytest.raises(ValueError):
        RoutingModel("zipf")
    with pytest.raises(ValueError):
        RoutingModel("sampled", 0.0)
