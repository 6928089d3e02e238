"""The engine's job list (paper_2503_09716_b200.schedule) vs the reference planner's own DAGs.

Golden DAGs were produced by /root/reference's moe_planner.build_forward_dag /
build_layer_dag (offload_dag.py:495-533) by tests/golden/make_golden.py.  Parity target
(SURVEY.md §8c engine target 1): identical node list (kind, resource, label, layer, tokens, seqs,
bytes, duration) and identical edge set, and the same critical path (plan_search.py:57-59)."""

import glob
import json
import math
import os

import pytest

from paper_2503_09716_b200.planner import (BatchingPlan, ModelSpec, WorkloadSpec, footprint, load_profile_document)
from paper_2503_09716_b200.schedule import (build_schedule, even_split, latency_from_curves, split_cap)

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "schedule_*.json")))


def _load(path):
    with open(path) as f:
        return json.load(f)


def _rebuild(doc):
    spec = ModelSpec.from_document(doc["model"])
    hw, curves = load_profile_document(doc["profile"])
    w = doc["workload"]
    wl = WorkloadSpec(w["prompt_len"], w["decode_len"], w["num_sequences"], w["phase"])
    plan = BatchingPlan.from_document(doc["plan"])
    if doc.get("layer_index") is not None:
        return build_schedule(spec, hw, latency_from_curves(curves), wl, plan, layers=[doc["layer_index"]],
                              serialize=False)
    return build_schedule(spec, hw, latency_from_curves(curves), wl, plan, expert_counts=doc["expert_tokens"])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_schedule_matches_reference_dag(path):
    doc = _load(path)
    ref = doc["dag"]
    sch = _rebuild(doc)
    assert len(sch.jobs) == len(ref["nodes"])
    for j, n in zip(sch.jobs, ref["nodes"]):
        assert (j.id, j.kind, j.resource, j.label, j.layer, j.tokens, j.seqs) == (
            n["id"], n["kind"], n["resource"], n["label"], n["layer"], n["tokens"], n["seqs"])
        assert j.nbytes == n["nbytes"]
        assert math.isclose(j.duration, n["duration"], rel_tol=1e-12, abs_tol=0.0)
    assert sorted(map(tuple, ref["edges"])) == sorted(sch.edges)
    assert (sch.entry, sch.exit) == (ref["entry"], ref["exit"])
    if doc.get("layer_index") is None:
        assert math.isclose(sch.critical_path(), doc["critical_path"], rel_tol=1e-12)


def test_golden_cases_present():
    names = {os.path.basename(p) for p in GOLDEN}
    assert "schedule_mixtral_a5000_searched.json" in names  # the 1,040-node plan of SURVEY §8a8
    assert len(GOLDEN) >= 6


def test_mixtral_searched_plan_shape():
    doc = _load(os.path.join(os.path.dirname(__file__), "golden", "schedule_mixtral_a5000_searched.json"))
    sch = _rebuild(doc)
    assert len(sch.jobs) == 1040  # hand-checked 17*32 + 15*33 - 1 + 2
    kinds = {}
    for j in sch.jobs:
        kinds[j.kind] = kinds.get(j.kind, 0) + 1
    assert kinds["attn_mech_cpu"] == 32 and kinds["router"] == 32


def test_resident_policy_drops_kv_traffic():
    doc = _load(os.path.join(os.path.dirname(__file__), "golden", "schedule_tinymixtral_b200_resident_weights.json"))
    spec = ModelSpec.from_document(doc["model"])
    hw, curves = load_profile_document(doc["profile"])
    w = doc["workload"]
    wl = WorkloadSpec(w["prompt_len"], w["decode_len"], w["num_sequences"], w["phase"])
    plan = BatchingPlan.from_document(doc["plan"])
    off = build_schedule(spec, hw, latency_from_curves(curves), wl, plan)
    res = build_schedule(spec, hw, latency_from_curves(curves), wl, plan, kv_policy="resident")
    k_off = [j.kind for j in off.jobs]
    k_res = [j.kind for j in res.jobs]
    assert "kv_copy_in" in k_off and "kv_copy_in" not in k_res and "kv_copy_out" not in k_res
    assert [k for k in k_off if not k.startswith("kv_copy")] == k_res
    fp = footprint(spec, hw, wl, plan, "resident")
    assert fp.s_kv_cpu == 0 and fp.s_kv_gpu == plan.B * wl.max_context * spec.kv_bytes_per_token_layer * spec.num_layers


def test_even_split_and_split_cap():
    assert even_split(10, 4) == [3, 3, 2, 2]
    assert even_split(8 * 6, 160)[:48] == [1] * 48 and sum(even_split(48, 160)) == 48
    assert split_cap(10, 4) == [4, 4, 2] and split_cap(0, 4) == [] and split_cap(8, 4) == [4, 4]


def test_serialized_resource_chains_are_in_submission_order():
    doc = _load(os.path.join(os.path.dirname(__file__), "golden", "schedule_tiny_decode_omega05.json"))
    sch = _rebuild(doc)
    es = set(sch.edges)
    for r in ("gpu_compute", "htod_link", "dtoh_link", "cpu_compute"):
        ids = [j.id for j in sch.jobs if j.resource == r]
        for u, v in zip(ids, ids[1:]):
            assert (u, v) in es
