"""The scheduler's plan search (paper_2503_09716_b200.plan_search) vs the reference planner.

1. forward_time (streaming critical path) == the critical path of the materialized schedule
   (schedule.build_schedule, itself golden-equal to the reference DAG) on every golden schedule and
   on a sweep of plans;
2. search / model_based_baseline winners, candidate counts and skip tallies == the reference's own
   search (plan_search.py:169-314) on tests/golden/search_*.json (tests/golden/make_golden_search.py).
"""

import glob
import json
import math
import os
import time

import pytest

from paper_2503_09716_b200.plan_search import (SearchSpace, enumerate_candidates, forward_time,
                                               model_based_baseline, search)
from paper_2503_09716_b200.planner import BatchingPlan, ModelSpec, WorkloadSpec, load_profile_document
from paper_2503_09716_b200.schedule import build_schedule, latency_from_curves

HERE = os.path.join(os.path.dirname(__file__), "golden")
SCHEDULES = sorted(glob.glob(os.path.join(HERE, "schedule_*.json")))
SEARCHES = sorted(glob.glob(os.path.join(HERE, "search_*.json")))


def _inputs(doc):
    spec = ModelSpec.from_document(doc["model"])
    hw, curves = load_profile_document(doc["profile"])
    w = doc["workload"]
    wl = WorkloadSpec(w["prompt_len"], w["decode_len"], w["num_sequences"], w["phase"])
    return spec, hw, latency_from_curves(curves), wl


@pytest.mark.parametrize("path", SCHEDULES, ids=[os.path.basename(p) for p in SCHEDULES])
def test_forward_time_equals_schedule_critical_path(path):
    doc = json.load(open(path))
    if doc.get("layer_index") is not None:
        pytest.skip("single-layer fixture")
    spec, hw, lat, wl = _inputs(doc)
    plan = BatchingPlan.from_document(doc["plan"])
    t = forward_time(spec, hw, lat, wl, plan, expert_counts=doc["expert_tokens"])
    assert math.isclose(t, doc["critical_path"], rel_tol=1e-12)


def test_forward_time_sweep_matches_build_schedule():
    doc = json.load(open(os.path.join(HERE, "search_tiny_decode.json")))
    spec, hw, lat, wl = _inputs(doc)
    n = 0
    for phase in ("decode", "prefill"):
        w = wl.with_phase(phase)
        for plan in enumerate_candidates(spec, hw, w, SearchSpace(b_a_grid=(16, 64), b_e_grid=(256, 4096),
                                                                  omega_grid=(0.0, 0.3, 0.5),
                                                                  s_expert_slots_grid=(2, 8))):
            ref = build_schedule(spec, hw, lat, w, plan).critical_path()
            assert math.isclose(forward_time(spec, hw, lat, w, plan), ref, rel_tol=1e-12), plan
            n += 1
    assert n > 50


@pytest.mark.parametrize("path", SEARCHES, ids=[os.path.basename(p) for p in SEARCHES])
def test_search_matches_reference(path):
    doc = json.load(open(path))
    spec, hw, lat, wl = _inputs(doc)
    wl = wl.with_phase(doc["phase"])
    space = SearchSpace.from_document(doc["space"])
    skips = {}
    assert sum(1 for _ in enumerate_candidates(spec, hw, wl, space, skip_counts=skips)) == doc["candidates"]
    assert skips == doc["skips"]
    t0 = time.time()
    best = search(spec, hw, lat, wl, space)
    dt = time.time() - t0
    assert best.plan == BatchingPlan.from_document(doc["best"]["plan"])
    assert math.isclose(best.t_forward, doc["best"]["t_forward"], rel_tol=1e-12)
    base = model_based_baseline(spec, hw, lat, wl)
    assert base.plan == BatchingPlan.from_document(doc["baseline"]["plan"])
    assert math.isclose(base.throughput, doc["baseline"]["throughput"], rel_tol=1e-12)
    print(f"{doc['name']}: {dt:.2f} s here vs {doc['reference_search_seconds']:.2f} s in the reference")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tiny-mixtral", "tiny-deepseek-v2"])
def test_measured_profile_feeds_search(name):
    """profiler.profile_engine measures every GPU module kind on the engine's kernels and emits the
    reference's profile schema (monotone tables, hw_profile.py:117-142); the search runs on it."""
    from paper_2503_09716_b200.configs import get_arch
    from paper_2503_09716_b200.profiler import profile_engine

    arch = get_arch(name)
    doc = profile_engine(arch, token_grid=[1, 2, 8, 32, 64], ctx_grid=(16, 64), reps=2)
    kinds = {t["module_kind"] for t in doc["latency_tables"]}
    assert kinds == {"pre_attention", "attention_mechanism_gpu", "post_attention", "router", "expert"}
    for t in doc["latency_tables"]:
        by_ctx = {}
        for tok, ctx, sec in t["entries"]:
            assert sec > 0
            by_ctx.setdefault(ctx, []).append((tok, sec))
        for pts in by_ctx.values():
            pts.sort()
            assert len(pts) >= 2 and all(a[1] <= b[1] for a, b in zip(pts, pts[1:]))
    hw, curves = load_profile_document(doc)
    assert hw.bw_htod > 1e9 and hw.m_g > 1e10
    spec = ModelSpec.from_document(arch.model_spec_document())
    space = SearchSpace(b_a_grid=(16, 64), b_e_grid=(256,), omega_grid=(0.0,), s_expert_slots_grid=(2,),
                        s_params_fracs=(0.0, 1.0))
    best = search(spec, hw, latency_from_curves(curves), WorkloadSpec(64, 32, 10_000), space)
    assert best.throughput > 0
    # per-module peak memory: every module kind, at every latency point, at least
    # the engine buffers it touches; the expert module's fitted per-row bytes are its x_perm, h_ffn
    # and y_perm rows (no transient allocation inside the grouped GEMMs)
    mkinds = {t["module_kind"]: t["entries"] for t in doc["memory_tables"]}
    assert set(mkinds) == kinds
    for t in doc["latency_tables"]:
        assert [e[:2] for e in mkinds[t["module_kind"]]] == [e[:2] for e in t["entries"]]
        assert all(e[2] > 0 for e in mkinds[t["module_kind"]])
    co = doc["activation_coefficients"]
    assert co["expert_activation_bytes_per_token"] == 2 * (2 * arch.hidden + arch.moe_ffn)
    assert co["attn_activation_bytes_per_token"] >= 2 * arch.hidden
    assert co["attn_activation_bytes_per_ctx_token"] == 0.0  # paged kernels: nothing per context token
    mspec = ModelSpec.from_document({**arch.model_spec_document(), **co})
    assert search(mspec, hw, latency_from_curves(curves), WorkloadSpec(64, 32, 10_000), space).throughput > 0


def test_activation_coefficients_fit():
    """The fit of profiler.activation_coefficients on a hand-made memory table: slopes per token
    (max over the attention modules), per context token per sequence, per routed expert row."""
    from paper_2503_09716_b200.profiler import activation_coefficients

    doc = {"memory_tables": [
        {"module_kind": "pre_attention", "entries": [[1, 0, 100 + 10], [64, 0, 100 + 640]]},
        {"module_kind": "post_attention", "entries": [[1, 0, 30], [64, 0, 30 * 64]]},
        {"module_kind": "attention_mechanism_gpu",
         "entries": [[1, 16, 8 + 16 * 2], [1, 64, 8 + 64 * 2], [64, 16, 64 * (8 + 16 * 2)], [64, 64, 64 * (8 + 64 * 2)]]},
        {"module_kind": "router", "entries": [[1, 0, 5], [64, 0, 320]]},
        {"module_kind": "expert", "entries": [[1, 0, 7 + 1000], [64, 0, 64 * 7 + 1000]]}]}
    co = activation_coefficients(doc)
    assert co == {"attn_activation_bytes_per_token": 40.0, "attn_activation_bytes_per_ctx_token": 2.0,
                  "expert_activation_bytes_per_token": 7.0}
