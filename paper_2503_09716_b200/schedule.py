"""The module-based batching job list: what the engine issues, in which order, on which stream.

This is the B200 engine's own builder of the schedule the reference encodes as its execution DAG
(reference: pkg/src/moe_planner/offload_dag.py:240-492 `_build_graph`, :536-564
`serialize_resources`; plan_search.py:43-59 critical path).  Job kinds, labels, launch shapes
(tokens / seqs / bytes), data + buffer-recycling edges and submission order are identical to
the reference for the same (model, workload, plan, routing counts) — tests/test_schedule.py
checks that against golden DAGs produced by the reference itself.

Resource -> B200 mapping: gpu_compute -> the compute stream, htod_link -> the H2D copy stream,
dtoh_link -> the D2H copy stream, cpu_compute -> a host worker; a serialized resource chain is
in-order stream semantics and a cross-resource edge is a cudaEvent wait.

kv_policy="resident" (B200 extension) keeps KV in HBM, so the KV copy-in jobs disappear and the
new-KV copy-out jobs disappear with them; everything else is unchanged.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Callable, Sequence

from .planner import BatchingPlan, Hardware, LatencyCurve, ModelSpec, WorkloadSpec, footprint, placement, validate

GPU, CPU, HTOD, DTOH = "gpu_compute", "cpu_compute", "htod_link", "dtoh_link"
RESOURCE_OF = {
    "weight_copy": HTOD, "kv_copy_in": HTOD, "kv_copy_out": DTOH, "pre_attention": GPU, "attn_mech_gpu": GPU,
    "attn_mech_cpu": CPU, "post_attention": GPU, "router": GPU, "expert_compute": GPU, "barrier": None,
}
# schedule job kind -> profiling module kind (hw_profile.py:52-58)
MODULE_OF = {"pre_attention": "pre_attention", "attn_mech_gpu": "attention_mechanism_gpu",
             "attn_mech_cpu": "attention_mechanism_cpu", "post_attention": "post_attention",
             "router": "router", "expert_compute": "expert"}


class InfeasibleSchedule(ValueError):
    pass


@dataclass(frozen=True)
class Job:
    id: int
    kind: str
    resource: str | None
    duration: float
    label: str
    layer: int = -1
    tokens: int = 0
    seqs: int = 0
    nbytes: float = 0.0


@dataclass
class Schedule:
    jobs: list
    edges: list
    entry: int
    exit: int

    def preds(self) -> list[list[int]]:
        p = [[] for _ in self.jobs]
        for u, v in self.edges:
            p[v].append(u)
        return p

    def succs(self) -> list[list[int]]:
        s = [[] for _ in self.jobs]
        for u, v in self.edges:
            s[u].append(v)
        return s

    def topo(self) -> list[int]:
        indeg = [0] * len(self.jobs)
        for _, v in self.edges:
            indeg[v] += 1
        succ = self.succs()
        stack = [i for i, d in enumerate(indeg) if d == 0]
        out = []
        while stack:
            u = stack.pop()
            out.append(u)
            for v in succ[u]:
                indeg[v] -= 1
                if indeg[v] == 0:
                    stack.append(v)
        if len(out) != len(self.jobs):
            raise ValueError("schedule contains a cycle")
        return out

    def serialized(self) -> "Schedule":
        """Chain same-resource jobs by id = submission order (offload_dag.py:536-564)."""
        have = set(self.edges)
        edges = list(self.edges)
        last: dict[str, int] = {}
        for j in self.jobs:
            if j.resource is None:
                continue
            if j.resource in last and (last[j.resource], j.id) not in have:
                have.add((last[j.resource], j.id))
                edges.append((last[j.resource], j.id))
            last[j.resource] = j.id
        out = Schedule(self.jobs, edges, self.entry, self.exit)
        out.topo()
        return out

    def finish_times(self) -> list[float]:
        preds = self.preds()
        dp = [0.0] * len(self.jobs)
        for v in self.topo():
            start = 0.0
            for u in preds[v]:
                if dp[u] > start:
                    start = dp[u]
            dp[v] = start + self.jobs[v].duration
        return dp

    def critical_path(self) -> float:
        return self.finish_times()[self.exit]

    def to_json(self) -> str:
        return json.dumps({"entry": self.entry, "exit": self.exit,
                           "nodes": [{"id": j.id, "kind": j.kind, "resource": j.resource, "duration": j.duration,
                                      "label": j.label} for j in self.jobs],
                           "edges": [list(e) for e in self.edges]}, indent=2, sort_keys=True)

    def launches(self, kinds: Sequence[str] | None = None) -> list[Job]:
        return [j for j in self.jobs if j.resource is not None and (kinds is None or j.kind in kinds)]


def even_split(total: int, buckets: int) -> list[int]:
    """Floor share everywhere, remainder to the leading buckets (offload_dag.py:173-177)."""
    q, r = divmod(total, buckets)
    return [q + (i < r) for i in range(buckets)]


def split_cap(n: int, cap: int) -> list[int]:
    """Greedy pieces of at most `cap` (micro-batches / expert chunks, offload_dag.py:221-237)."""
    full, rem = divmod(n, cap)
    return [cap] * full + ([rem] if rem else [])


LatencyFn = Callable[[str, int, int], float]


def latency_from_curves(curves: Sequence[LatencyCurve]) -> LatencyFn:
    by_kind = {c.module_kind: c for c in curves}

    def lat(module_kind: str, tokens: int, context: int) -> float:
        if tokens < 1:
            raise ValueError("tokens must be >= 1")
        if module_kind not in by_kind:
            raise KeyError(f"no latency table for module kind {module_kind!r}")
        return by_kind[module_kind](tokens, context)

    return lat


def build_schedule(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec, plan: BatchingPlan,
                   phase: str | None = None, layers: Sequence[int] | None = None,
                   expert_counts: Sequence[Sequence[int]] | None = None, kv_policy: str = "offload",
                   serialize: bool = True) -> Schedule:
    """Job list for one forward pass over `layers` (default: all), see module docstring."""
    wl = wl.with_phase(phase or wl.phase)
    validate(spec, plan)
    fp = footprint(spec, hw, wl, plan, kv_policy)
    if not fp.feasible:
        raise InfeasibleSchedule(f"plan violates memory constraints (host_feasible={fp.host_feasible}, "
                                 f"gpu_feasible={fp.gpu_feasible})")
    layers = list(range(spec.num_layers)) if layers is None else list(layers)
    prefill = wl.phase == "prefill"
    tif = wl.tokens_per_seq_in_flight
    ctx = wl.prompt_len if prefill else wl.max_context
    kv = spec.kv_bytes_per_token_layer
    n_cpu, n_gpu = plan.cpu_sequences(), plan.gpu_sequences()
    if n_cpu > 0 and hw.cpu_attn_flops == 0:
        raise InfeasibleSchedule("plan routes attention to the CPU but no CPU attention rate is available")
    place = placement(spec, plan.s_params)
    slots = plan.s_expert // spec.expert_bytes
    batch_tokens = plan.B * tif
    stream_kv = kv_policy == "offload" and not prefill
    ring = 0
    if stream_kv and n_gpu > 0:
        slice_bytes = plan.b_a * ctx * kv
        spare = (hw.m_g - fp.gpu_total) + fp.s_kv_gpu
        ring = max(1, int(spare // slice_bytes))

    jobs: list[Job] = []
    edges: list[tuple[int, int]] = []
    seen: set[tuple[int, int]] = set()

    def edge(u: int, v: int) -> None:
        if (u, v) not in seen:
            seen.add((u, v))
            edges.append((u, v))

    def job(kind: str, duration: float, label: str, deps=(), **kw) -> int:
        i = len(jobs)
        jobs.append(Job(i, kind, RESOURCE_OF[kind], duration, label, **kw))
        for d in deps:
            edge(d, i)
        return i

    boundary: int | None = None
    dense_owner: int | None = None   # post-attention of the last uncached dense layer
    fetches: list[tuple[int, int]] = []  # (expert copy, its last consumer), global order
    kv_slices: list[tuple[int, int]] = []  # (kv copy-in, consuming mechanism)

    for li, layer in enumerate(layers):
        base = [boundary] if boundary is not None else []
        # ---- dense weights (single dense buffer) ----
        dense = None
        if layer >= place.dense_layers:
            dense = job("weight_copy", spec.dense_bytes_per_layer / hw.bw_htod, f"L{layer}/dense_copy", layer=layer,
                        nbytes=float(spec.dense_bytes_per_layer))
            if dense_owner is not None:
                edge(dense_owner, dense)
        cdeps = base + ([dense] if dense is not None else [])
        mechs: list[int] = []
        # ---- CPU attention share (issued first) ----
        if n_cpu > 0:
            nt = n_cpu * tif
            pre = job("pre_attention", latency("pre_attention", nt, ctx), f"L{layer}/pre_attn/cpu", cdeps,
                      layer=layer, tokens=nt, seqs=n_cpu)
            job("kv_copy_out", nt * kv / hw.bw_dtoh, f"L{layer}/kv_out/cpu", (pre,), layer=layer, nbytes=float(nt * kv))
            mechs.append(job("attn_mech_cpu", latency("attention_mechanism_cpu", nt, ctx), f"L{layer}/attn_cpu",
                             (pre,), layer=layer, tokens=nt, seqs=n_cpu))
        # ---- GPU attention micro-batches of <= b_a sequences ----
        for mb, s in enumerate(split_cap(n_gpu, plan.b_a)):
            nt = s * tif
            pre = job("pre_attention", latency("pre_attention", nt, ctx), f"L{layer}/pre_attn/mb{mb}", cdeps,
                      layer=layer, tokens=nt, seqs=s)
            mdeps = [pre]
            kin = None
            if stream_kv:
                kin = job("kv_copy_in", s * ctx * kv / hw.bw_htod, f"L{layer}/kv_in/mb{mb}", layer=layer,
                          nbytes=float(s * ctx * kv))
                if len(kv_slices) >= ring:
                    edge(kv_slices[-ring][1], kin)
                mdeps.append(kin)
            if kv_policy == "offload":
                job("kv_copy_out", nt * kv / hw.bw_dtoh, f"L{layer}/kv_out/mb{mb}", (pre,), layer=layer,
                    nbytes=float(nt * kv))
            mech = job("attn_mech_gpu", latency("attention_mechanism_gpu", nt, ctx), f"L{layer}/attn_gpu/mb{mb}",
                       mdeps, layer=layer, tokens=nt, seqs=s)
            mechs.append(mech)
            if kin is not None:
                kv_slices.append((kin, mech))
        # ---- post-attention barrier, router ----
        post = job("post_attention", latency("post_attention", batch_tokens, ctx), f"L{layer}/post_attn",
                   mechs if mechs else cdeps, layer=layer, tokens=batch_tokens, seqs=plan.B)
        if dense is not None:
            dense_owner = post
        router = job("router", latency("router", batch_tokens, ctx), f"L{layer}/router", (post,), layer=layer,
                     tokens=batch_tokens)
        # ---- experts, ascending index; copies recycle `slots` buffer slots ----
        counts = list(expert_counts[li]) if expert_counts is not None else even_split(batch_tokens * spec.top_k,
                                                                                         spec.experts_per_layer)
        if len(counts) != spec.experts_per_layer:
            raise ValueError("expert_tokens row length != experts_per_layer")
        cached = place.experts_per_layer[layer % spec.num_layers]
        computes: list[int] = []
        for e, n_e in enumerate(counts):
            cp = None
            if e >= cached:
                cp = job("weight_copy", spec.expert_bytes / hw.bw_htod, f"L{layer}/expert{e}_copy", layer=layer,
                         nbytes=float(spec.expert_bytes))
                if slots > 0 and len(fetches) >= slots:
                    edge(fetches[-slots][1], cp)
            last = router
            for j, chunk in enumerate(split_cap(n_e, plan.b_e)):
                last = job("expert_compute", latency("expert", chunk, ctx), f"L{layer}/expert{e}/chunk{j}",
                           [router] + ([cp] if cp is not None else []), layer=layer, tokens=chunk)
                computes.append(last)
            if cp is not None:
                fetches.append((cp, last))
        if li < len(layers) - 1:
            boundary = job("barrier", 0.0, f"L{layer}/boundary", computes, layer=layer)

    n = len(jobs)
    has_pred = [False] * n
    has_succ = [False] * n
    for u, v in edges:
        has_succ[u] = True
        has_pred[v] = True
    entry = job("barrier", 0.0, "entry")
    for i in range(n):
        if not has_pred[i]:
            edge(entry, i)
    exit_ = job("barrier", 0.0, "exit")
    for i in range(n):
        if not has_succ[i]:
            edge(i, exit_)
    sch = Schedule(jobs, edges, entry, exit_)
    sch.topo()
    return sch.serialized() if serialize else sch
