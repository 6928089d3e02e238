"""Batching-strategy search: the scheduler's choice of (B, b_a, b_e, omega, s_expert, s_params).

Same decisions as the reference planner (pkg/src/moe_planner/plan_search.py): candidates are the
grid product of `SearchSpace` (:122-166) enumerated in the same order with the same feasibility
filters (:169-238), each scored by forward throughput = tokens per forward / critical path of the
serialized forward schedule (:43-105), and the winner is the highest throughput with ties broken
toward the lexicographically smallest (B, b_a, b_e, omega, s_expert, s_params) (:77-79, 241-261).
`model_based_baseline` is the unified-batch baseline (:264-314).

What is B200-specific is the evaluator.  The reference materializes every candidate's DAG and runs
a topological DP over it (20-170 s per Mixtral search).  Here `forward_time` streams the schedule
instead: jobs are produced in submission order (= id order, which is also the serialization order
of each resource queue, offload_dag.py:536-564) and every data edge points to an earlier job, so a
job's earliest finish is known the moment it is produced:

    finish(j) = max(finish(data preds of j), finish(previous job on j's resource)) + duration(j)

and the critical path is the largest finish.  Latencies are memoized per (module, tokens) because
the context is fixed within one evaluation.  tests/test_plan_search.py checks forward_time against
schedule.build_schedule(...).critical_path() and the winners against the reference's own search.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Iterator, Sequence

from .planner import (BatchingPlan, Footprint, Hardware, ModelSpec, PlanError, WorkloadSpec, footprint,
                      largest_batch, placement, validate, MIN_EXPERT_SLOTS)
from .schedule import LatencyFn, even_split, split_cap


class EmptySearchSpace(RuntimeError):
    pass


def forward_time(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec, plan: BatchingPlan,
                 kv_policy: str = "offload", expert_counts: Sequence[Sequence[int]] | None = None) -> float:
    """Critical path of the serialized forward schedule build_schedule() would produce (seconds).
    Raises ValueError (PlanError / infeasible) exactly when build_schedule would."""
    validate(spec, plan)
    fp = footprint(spec, hw, wl, plan, kv_policy)
    if not fp.feasible:
        raise ValueError("plan violates memory constraints")
    prefill = wl.phase == "prefill"
    tif = wl.tokens_per_seq_in_flight
    ctx = wl.prompt_len if prefill else wl.max_context
    kv = spec.kv_bytes_per_token_layer
    n_cpu, n_gpu = plan.cpu_sequences(), plan.gpu_sequences()
    if n_cpu > 0 and hw.cpu_attn_flops == 0:
        raise ValueError("plan routes attention to the CPU but no CPU attention rate is available")
    place = placement(spec, plan.s_params)
    slots = plan.s_expert // spec.expert_bytes
    batch_tokens = plan.B * tif
    stream_kv = kv_policy == "offload" and not prefill
    ring = 0
    if stream_kv and n_gpu > 0:
        ring = max(1, int(((hw.m_g - fp.gpu_total) + fp.s_kv_gpu) // (plan.b_a * ctx * kv)))

    memo: dict[tuple[str, int], float] = {}

    def lat(kind: str, tokens: int) -> float:
        v = memo.get((kind, tokens))
        if v is None:
            v = memo[(kind, tokens)] = latency(kind, tokens, ctx)
        return v

    last = {"gpu_compute": 0.0, "cpu_compute": 0.0, "htod_link": 0.0, "dtoh_link": 0.0}
    end = 0.0

    def run(res: str, dur: float, ready: float) -> float:
        nonlocal end
        f = max(ready, last[res]) + dur
        last[res] = f
        if f > end:
            end = f
        return f

    GPU, CPU, HTOD, DTOH = "gpu_compute", "cpu_compute", "htod_link", "dtoh_link"
    boundary = 0.0
    dense_owner: float | None = None
    fetch_done: list[float] = []   # finish of the last consumer of each expert copy (global order)
    kv_mech: list[float] = []      # finish of the mechanism consuming each KV slice
    mb_sizes = split_cap(n_gpu, plan.b_a)
    n_layers = spec.num_layers
    for li in range(n_layers):
        dense = None
        if li >= place.dense_layers:
            dense = run(HTOD, spec.dense_bytes_per_layer / hw.bw_htod, dense_owner or 0.0)
        cready = max(boundary, dense or 0.0)
        mechs: list[float] = []
        if n_cpu > 0:
            nt = n_cpu * tif
            pre = run(GPU, lat("pre_attention", nt), cready)
            run(DTOH, nt * kv / hw.bw_dtoh, pre)
            mechs.append(run(CPU, lat("attention_mechanism_cpu", nt), pre))
        for s in mb_sizes:
            nt = s * tif
            pre = run(GPU, lat("pre_attention", nt), cready)
            mready = pre
            if stream_kv:
                rdy = kv_mech[-ring] if len(kv_mech) >= ring else 0.0
                kin = run(HTOD, s * ctx * kv / hw.bw_htod, rdy)
                mready = max(mready, kin)
            if kv_policy == "offload":
                run(DTOH, nt * kv / hw.bw_dtoh, pre)
            mech = run(GPU, lat("attention_mechanism_gpu", nt), mready)
            mechs.append(mech)
            if stream_kv:
                kv_mech.append(mech)
        post = run(GPU, lat("post_attention", batch_tokens), max(mechs) if mechs else cready)
        if dense is not None:
            dense_owner = post
        router = run(GPU, lat("router", batch_tokens), post)
        counts = (list(expert_counts[li]) if expert_counts is not None
                  else even_split(batch_tokens * spec.top_k, spec.experts_per_layer))
        cached = place.experts_per_layer[li % n_layers]
        layer_end = 0.0  # the layer boundary barrier: max over this layer's expert jobs
        for e, n_e in enumerate(counts):
            cp = None
            if e >= cached:
                rdy = fetch_done[-slots] if slots > 0 and len(fetch_done) >= slots else 0.0
                cp = run(HTOD, spec.expert_bytes / hw.bw_htod, rdy)
            ready = router if cp is None else max(router, cp)
            f = router
            for chunk in split_cap(n_e, plan.b_e):
                f = run(GPU, lat("expert", chunk), ready)
                layer_end = max(layer_end, f)
            if cp is not None:
                fetch_done.append(f)
        boundary = layer_end
    return end


def tokens_per_forward(wl: WorkloadSpec, B: int) -> int:
    return B * (wl.prompt_len if wl.phase == "prefill" else 1)


@dataclass(frozen=True)
class PlanEvaluation:
    plan: BatchingPlan
    phase: str
    t_forward: float
    throughput: float
    footprint: Footprint
    feasible: bool = True

    def sort_key(self) -> tuple:
        p = self.plan
        return (-self.throughput, p.B, p.b_a, p.b_e, p.omega, p.s_expert, p.s_params)


def evaluate_plan(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec, plan: BatchingPlan,
                  kv_policy: str = "offload") -> PlanEvaluation:
    """Score one plan (plan_search.py:82-105): infeasible plans come back with throughput 0."""
    fp = footprint(spec, hw, wl, plan, kv_policy)
    if not fp.feasible:
        return PlanEvaluation(plan, wl.phase, math.inf, 0.0, fp, False)
    try:
        t = forward_time(spec, hw, latency, wl, plan, kv_policy)
    except ValueError:
        return PlanEvaluation(plan, wl.phase, math.inf, 0.0, fp, False)
    return PlanEvaluation(plan, wl.phase, t, tokens_per_forward(wl, plan.B) / t, fp)


@dataclass(frozen=True)
class SearchSpace:
    b_a_grid: tuple = (16, 64, 256, 1024)
    b_e_grid: tuple = (256, 1024, 4096, 16384)
    omega_grid: tuple = tuple(round(0.1 * i, 1) for i in range(11))
    s_expert_slots_grid: tuple = (2, 4, 8, 32)
    s_params_fracs: tuple = (0.0, 0.25, 0.5, 0.75, 1.0)
    prefill_B_grid: tuple | None = None

    @classmethod
    def from_document(cls, d: dict) -> "SearchSpace":
        return cls(**{k: (tuple(v) if isinstance(v, list) else v) for k, v in d.items()})


def _powers_of_two(lo: int, hi: int) -> list[int]:
    out, v = [], 1
    while v <= hi:
        if v >= lo:
            out.append(v)
        v *= 2
    return out


def enumerate_candidates(spec: ModelSpec, hw: Hardware, wl: WorkloadSpec, space: SearchSpace,
                         kv_policy: str = "offload", skip_counts: dict | None = None) -> Iterator[BatchingPlan]:
    """Every feasible plan of the grid product, in the reference's order (plan_search.py:169-238)."""
    skips = skip_counts if skip_counts is not None else {}

    def skip(reason: str) -> None:
        skips[reason] = skips.get(reason, 0) + 1

    yielded = 0
    for omega in space.omega_grid:
        if omega > 0 and hw.cpu_attn_flops == 0:
            skip("cpu_unavailable")
            continue
        for b_a in space.b_a_grid:
            for b_e in space.b_e_grid:
                for slots in space.s_expert_slots_grid:
                    tmpl = BatchingPlan(1, b_a, b_e, omega, slots * spec.expert_bytes, 0)
                    try:
                        b_max = largest_batch(spec, hw, wl, tmpl, kv_policy)
                    except ValueError:
                        skip("no_feasible_B")
                        continue
                    if wl.phase == "decode":
                        b_grid = [b_max]
                    elif space.prefill_B_grid is not None:
                        b_grid = [x for x in space.prefill_B_grid if x <= b_max]
                        if not b_grid:
                            skip("no_feasible_B")
                    else:
                        b_grid = _powers_of_two(1, b_max)
                    for B in b_grid:
                        if omega < 1.0 and b_a > math.ceil((1.0 - omega) * B):
                            skip("b_a_exceeds_gpu_share")
                            continue
                        base = replace(tmpl, B=B)
                        fp = footprint(spec, hw, wl, base, kv_policy)
                        if not fp.feasible:
                            skip("infeasible")
                            continue
                        spare = hw.m_g - fp.gpu_total
                        for frac in space.s_params_fracs:
                            plan = replace(base, s_params=min(spec.model_bytes, int(frac * spare)))
                            try:
                                validate(spec, plan)
                            except PlanError:
                                skip("invalid_plan")
                                continue
                            if not footprint(spec, hw, wl, plan, kv_policy).feasible:
                                skip("infeasible")
                                continue
                            yielded += 1
                            yield plan
    if yielded == 0:
        raise EmptySearchSpace(f"no feasible candidate in the search space (skips: {skips})")


def search(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec, space: SearchSpace | None = None,
           kv_policy: str = "offload") -> PlanEvaluation:
    """Highest-throughput feasible plan; ties -> smallest (B, b_a, b_e, omega, s_expert, s_params)."""
    space = space or SearchSpace()
    best: PlanEvaluation | None = None
    for plan in enumerate_candidates(spec, hw, wl, space, kv_policy):
        ev = evaluate_plan(spec, hw, latency, wl, plan, kv_policy)
        if ev.feasible and (best is None or ev.sort_key() < best.sort_key()):
            best = ev
    if best is None:
        raise EmptySearchSpace("every candidate evaluated infeasible")
    return best


def model_based_baseline(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec,
                         s_params_fracs: Sequence[float] = (0.0, 0.25, 0.5, 0.75, 1.0),
                         kv_policy: str = "offload") -> PlanEvaluation:
    """Unified-batch baseline (plan_search.py:264-314): B = b_a, b_e = B*k, omega = 0, feasible in
    both phases, B doubled while it fits."""
    s_expert = MIN_EXPERT_SLOTS * spec.expert_bytes
    phases = [wl.with_phase("prefill")] + ([wl.with_phase("decode")] if wl.decode_len > 0 else [])

    def ok(p: BatchingPlan) -> bool:
        return all(footprint(spec, hw, w, p, kv_policy).feasible for w in phases)

    best: PlanEvaluation | None = None
    B = 1
    while True:
        p0 = BatchingPlan(B, B, B * spec.top_k, 0.0, s_expert, 0)
        if not ok(p0):
            break
        spare = min(hw.m_g - footprint(spec, hw, w, p0, kv_policy).gpu_total for w in phases)
        for frac in s_params_fracs:
            p = replace(p0, s_params=min(spec.model_bytes, int(frac * spare)))
            if not ok(p):
                continue
            ev = evaluate_plan(spec, hw, latency, wl, p, kv_policy)
            if ev.feasible and (best is None or ev.sort_key() < best.sort_key()):
                best = ev
        B *= 2
    if best is None:
        raise EmptySearchSpace("no unified batch size fits in memory")
    return best
