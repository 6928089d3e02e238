"""The engine's host-side planning interface vs the reference memory model (golden rows produced
by moe_planner.check_constraints / max_feasible_B / cache_placement, memory_model.py:147-277)."""

import json
import os

import pytest

from paper_2503_09716_b200.configs import ARCHS, MIXTRAL_8X7B
from paper_2503_09716_b200.planner import (BatchingPlan, Hardware, ModelSpec, PlanError, SpecError, WorkloadSpec,
                                           footprint, largest_batch, load_plan, placement, validate)

with open(os.path.join(os.path.dirname(__file__), "golden", "memory_model.json")) as f:
    GOLD = json.load(f)


def _hw(d):
    return Hardware(**{k: d[k] for k in ("m_g", "m_c", "bw_htod", "bw_dtoh", "gpu_peak_flops", "gpu_mem_bw",
                                         "gpu_launch_overhead", "cpu_attn_flops")})


@pytest.mark.parametrize("i", range(len(GOLD["rows"])))
def test_memory_model_rows(i):
    row = GOLD["rows"][i]
    spec = ModelSpec.from_document(row["model"])
    hw = _hw(row["hw"])
    p, d, n, phase = row["workload"]
    wl = WorkloadSpec(p, d, n, phase)
    tmpl = BatchingPlan(*row["template"])
    if row["max_feasible_B"] is None:
        with pytest.raises(ValueError):
            largest_batch(spec, hw, wl, tmpl)
    else:
        assert largest_batch(spec, hw, wl, tmpl) == row["max_feasible_B"]
    plan = BatchingPlan(*row["plan"])
    fp = footprint(spec, hw, wl, plan)
    assert [fp.s_kv_cpu, fp.s_kv_gpu, fp.s_is, fp.host_total, fp.gpu_total, fp.host_feasible,
            fp.gpu_feasible] == row["footprint"]
    pl = placement(spec, plan.s_params)
    assert [pl.dense_layers, list(pl.experts_per_layer), pl.cached_bytes, pl.uncached_expert_count] == row["placement"]
    assert plan.cpu_sequences() == row["cpu_sequences"]


def test_cpu_sequences_bankers_rounding():
    for B, om, expect in GOLD["cpu_sequences"]:
        assert BatchingPlan(B, 1, 1, om, 0, 0).cpu_sequences() == expect


def test_reference_golden_vectors():
    """Known answers pinned by the reference's own tests (test_memory_model.py:59-63,96-99;
    test_model_catalog.py:61-71)."""
    import math

    mix = ModelSpec.from_document(MIXTRAL_8X7B.model_spec_document())
    wl = WorkloadSpec(512, 256, 10_000, "decode")
    assert wl.max_context * mix.kv_bytes_per_token_layer * mix.num_layers == 100_663_296  # KV bytes / seq
    assert 64 * wl.max_context * mix.kv_bytes_per_token_layer == 201_326_592  # b_a=64 KV slice
    assert mix.expert_bytes == 352_321_536
    assert math.isclose(mix.num_layers * mix.experts_per_layer * mix.expert_bytes / 1e9, 90.2, rel_tol=1e-3)


def test_plan_document_round_trip(tmp_path):
    plan = BatchingPlan(1620, 256, 1024, 0.6, 8 * 352_321_536, 20_000_000_000)
    doc = {"plan": plan.to_document(), "phase": "decode", "t_forward": 1.0, "throughput": 1.0, "feasible": True}
    p = tmp_path / "plan.json"
    p.write_text(json.dumps(doc))
    assert load_plan(str(p)) == plan
    assert load_plan(plan.to_document()) == plan
    with pytest.raises(ValueError):
        load_plan({"B": 1})


def test_validate_errors_name_the_field():
    spec = ModelSpec.from_document(MIXTRAL_8X7B.model_spec_document())
    with pytest.raises(PlanError) as e:
        validate(spec, BatchingPlan(10, 11, 1, 0.0, 2 * spec.expert_bytes, 0))
    assert e.value.field == "b_a"
    with pytest.raises(PlanError) as e:
        validate(spec, BatchingPlan(10, 1, 1, 0.25, 2 * spec.expert_bytes, 0))
    assert e.value.field == "omega"
    with pytest.raises(PlanError) as e:
        validate(spec, BatchingPlan(10, 1, 1, 0.0, spec.expert_bytes, 0))
    assert e.value.field == "s_expert"
    validate(spec, BatchingPlan(10, 1, 1, 0.0, 0, spec.model_bytes))  # resident: no slots needed


def test_spec_validation():
    doc = dict(MIXTRAL_8X7B.model_spec_document())
    doc["top_k"] = 99
    with pytest.raises(SpecError):
        ModelSpec.from_document(doc)
    doc = dict(MIXTRAL_8X7B.model_spec_document())
    del doc["expert_bytes"]
    with pytest.raises(SpecError):
        ModelSpec.from_document(doc)


@pytest.mark.parametrize("name", sorted(ARCHS))
def test_arch_documents_load(name):
    a = ARCHS[name]
    spec = ModelSpec.from_document(a.model_spec_document())
    assert spec.num_layers == a.layers and spec.top_k == a.top_k
    assert a.total_params() > 0


def test_resident_plan_fits_b200():
    from paper_2503_09716_b200.engine import resident_plan

    plan = resident_plan(MIXTRAL_8X7B, 512, 256, hbm_bytes=183_359 << 20)
    spec = ModelSpec.from_document(MIXTRAL_8X7B.model_spec_document())
    kv = plan.B * 768 * spec.kv_bytes_per_token_layer * spec.num_layers
    assert spec.model_bytes + kv <= (183_359 << 20) - (12 << 30)
    assert plan.B >= 700
