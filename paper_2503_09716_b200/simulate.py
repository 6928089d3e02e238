"""Event-driven model of one forward pass of a batching plan: the reference's engine simulator
(pkg/src/moe_planner/exec_sim.py:161-344, `simulate_plan` / `SimReport`; routing stand-in
`RoutingModel` / `sample_routing` :41-81; `compare_with_estimate` :347-360), run over this
framework's schedule (`schedule.build_schedule`, golden-equal to the reference `_build_graph`).

The engine executes that same schedule on CUDA streams; `Engine.trace_step` measures it and reports
the same fields.  The simulator is the model the measurement is compared against
(tests/test_simulate.py pins it to the reference on golden reports; tests/test_sim_parity_gpu.py
runs the engine with the simulator's routing counts and its measured latency tables).

Semantics (as the reference): four single-server resources (gpu_compute, cpu_compute, htod_link,
dtoh_link) serve their jobs strictly in submission (id) order with head-of-line blocking; a job
starts at max(all predecessors finished, its server free); barrier jobs finish when ready.  GPU
occupancy = static reservations (cached parameters, expert slots, the dense buffer, the
accumulated batch's hidden states) + attention / expert activations while they run + each KV
slice from the start of its copy-in until its attention finishes; releases sort before acquires at
equal times.  `oom_flag` = peak > m_g.  Per-expert token groups larger than b_e split into extra
chunk jobs (the schedule does this).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import IO, Sequence

import numpy as np

from .planner import BatchingPlan, Hardware, ModelSpec, WorkloadSpec
from .schedule import GPU, HTOD, DTOH, LatencyFn, build_schedule, even_split

RESOURCES = ("gpu_compute", "cpu_compute", "htod_link", "dtoh_link")


@dataclass(frozen=True)
class RoutingModel:
    """Per-expert token counts of a MoE layer (exec_sim.py:41-59): "even" = even_split; "sampled" =
    symmetric Dirichlet(concentration) expert probabilities, multinomial counts, seeded per
    (seed, layer)."""

    mode: str = "even"
    concentration: float = 1.0
    seed: int = 0

    def __post_init__(self) -> None:
        if self.mode not in ("even", "sampled"):
            raise ValueError(f"unknown routing mode {self.mode!r}")
        if self.concentration <= 0:
            raise ValueError("concentration must be positive")


def sample_routing(spec: ModelSpec, tokens: int, routing: RoutingModel, layer: int) -> list[int]:
    """Counts per expert for one layer, summing to tokens * top_k (exec_sim.py:61-81; numpy's
    PCG64 stream seeded with [seed, layer], so the counts equal the reference's draw)."""
    if tokens < 1:
        raise ValueError("tokens must be >= 1")
    total = tokens * spec.top_k
    if routing.mode == "even":
        return even_split(total, spec.experts_per_layer)
    rng = np.random.default_rng([routing.seed, layer])
    probs = rng.dirichlet(np.full(spec.experts_per_layer, routing.concentration))
    return [int(c) for c in rng.multinomial(total, probs)]


@dataclass(frozen=True)
class SimReport:
    """exec_sim.py:84-110."""

    makespan: float
    busy: dict
    idle_fraction: dict
    bytes_htod: float
    bytes_dtoh: float
    peak_gpu_bytes: float
    expert_tokens: tuple
    mean_tokens_per_expert: float
    throughput: float
    oom_flag: bool

    def to_document(self) -> dict:
        return {"makespan": self.makespan, "busy": dict(self.busy), "idle_fraction": dict(self.idle_fraction),
                "bytes_htod": self.bytes_htod, "bytes_dtoh": self.bytes_dtoh, "peak_gpu_bytes": self.peak_gpu_bytes,
                "expert_tokens": [list(r) for r in self.expert_tokens],
                "mean_tokens_per_expert": self.mean_tokens_per_expert, "throughput": self.throughput,
                "oom_flag": self.oom_flag}

    def to_json(self) -> str:
        return json.dumps(self.to_document(), indent=2, sort_keys=True)


def _activation_bytes(spec: ModelSpec, wl: WorkloadSpec, job) -> float:
    """Transient GPU bytes of a running attention / expert job (exec_sim.py:139-158)."""
    context = wl.prompt_len if wl.phase == "prefill" else wl.max_context
    if job.kind == "attn_mech_gpu":
        return job.tokens * spec.attn_activation_per_token + job.seqs * context * spec.attn_activation_bytes_per_ctx_token
    if job.kind == "expert_compute":
        return job.tokens * spec.expert_activation_per_token
    return 0.0


def simulate_plan(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec, plan: BatchingPlan,
                  routing: RoutingModel = RoutingModel(), phase: str | None = None, kv_policy: str = "offload",
                  trace_stream: IO[str] | None = None, expert_counts: Sequence[Sequence[int]] | None = None
                  ) -> SimReport:
    """Run the plan's job list over the four resources.  `expert_counts` (per layer, per expert)
    overrides the routing model, e.g. with the counts an engine step actually routed."""
    wl = wl.with_phase(phase or wl.phase)
    batch_tokens = plan.B * wl.tokens_per_seq_in_flight
    counts = ([list(map(int, r)) for r in expert_counts] if expert_counts is not None else
              [sample_routing(spec, batch_tokens, routing, l) for l in range(spec.num_layers)])
    sch = build_schedule(spec, hw, latency, wl, plan, expert_counts=counts, kv_policy=kv_policy, serialize=False)
    jobs = sch.jobs
    n = len(jobs)
    preds, succs = sch.preds(), sch.succs()
    static_bytes = float(plan.s_params + plan.s_expert + spec.dense_bytes_per_layer
                         + plan.B * wl.tokens_per_seq_in_flight * spec.hidden_bytes_per_token)
    # KV slice held from its copy-in start until the consuming attention finishes
    kv_consumer: dict[int, int] = {}
    kv_release: dict[int, float] = {}
    for j in jobs:
        if j.kind == "kv_copy_in":
            for s in succs[j.id]:
                if jobs[s].kind == "attn_mech_gpu":
                    kv_consumer[j.id] = s
                    kv_release[s] = kv_release.get(s, 0.0) + j.nbytes
                    break
    # FIFO + head-of-line blocking on a server == start after the previous job of the same resource
    # (submission order = id order) and after all predecessors: evaluate in topological order of the
    # DAG plus those chains
    order_preds = [list(p) for p in preds]
    last: dict[str, int] = {}
    queue: dict[str, list[int]] = {r: [] for r in RESOURCES}
    for j in jobs:
        if j.resource is not None:
            if j.resource in last:
                order_preds[j.id].append(last[j.resource])
            last[j.resource] = j.id
            queue[j.resource].append(j.id)
    indeg = [len(p) for p in order_preds]
    out_edges: list[list[int]] = [[] for _ in range(n)]
    for v, ps in enumerate(order_preds):
        for u in ps:
            out_edges[u].append(v)
    start = [0.0] * n
    finish = [0.0] * n
    ready = [0.0] * n
    stack = [v for v in range(n) if indeg[v] == 0]
    done = 0
    while stack:
        v = stack.pop()
        done += 1
        j = jobs[v]
        t = 0.0
        for u in preds[v]:
            t = max(t, finish[u])
        ready[v] = t
        if j.resource is None:
            start[v] = finish[v] = t
        else:
            prev = [u for u in order_preds[v][len(preds[v]):]]
            s = max([t] + [finish[u] for u in prev])
            start[v], finish[v] = s, s + j.duration
        for w in out_edges[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                stack.append(w)
    if done != n:
        raise RuntimeError("simulation deadlocked; schedule or queues inconsistent")
    busy = {r: 0.0 for r in RESOURCES}
    bytes_htod = bytes_dtoh = 0.0
    deltas: list[tuple[float, int, float]] = []
    for r in RESOURCES:
        for v in queue[r]:
            j = jobs[v]
            busy[r] += j.duration
            if r == HTOD:
                bytes_htod += j.nbytes
                if j.kind == "kv_copy_in" and v in kv_consumer:
                    deltas.append((start[v], 1, j.nbytes))
            elif r == DTOH:
                bytes_dtoh += j.nbytes
            if r == GPU:
                act = _activation_bytes(spec, wl, j)
                if act:
                    deltas.append((start[v], 1, act))
                    deltas.append((finish[v], 0, -act))
                if v in kv_release:
                    deltas.append((finish[v], 0, -kv_release[v]))
    makespan = max((finish[v] for v in range(n) if jobs[v].resource is not None), default=0.0)
    peak = level = static_bytes
    for _, _, d in sorted(deltas):
        level += d
        peak = max(peak, level)
    if trace_stream is not None:
        recs = []
        for v in range(n):
            j = jobs[v]
            for order, (action, t) in enumerate((("start", start[v]), ("finish", finish[v]))):
                recs.append((t, v, order, {"time": t, "node": v, "kind": j.kind, "resource": j.resource,
                                           "action": action}))
        for _, _, _, rec in sorted(recs, key=lambda e: (e[0], e[1], e[2])):
            trace_stream.write(json.dumps(rec, sort_keys=True) + "\n")
    flat = [c for row in counts for c in row]
    return SimReport(
        makespan=makespan, busy=busy,
        idle_fraction={r: (1.0 - busy[r] / makespan) if makespan > 0 else 0.0 for r in RESOURCES},
        bytes_htod=bytes_htod, bytes_dtoh=bytes_dtoh, peak_gpu_bytes=peak,
        expert_tokens=tuple(tuple(r) for r in counts), mean_tokens_per_expert=sum(flat) / len(flat),
        throughput=batch_tokens / makespan if makespan > 0 else math.inf, oom_flag=peak > hw.m_g)


def compare_with_estimate(spec: ModelSpec, hw: Hardware, latency: LatencyFn, wl: WorkloadSpec, plan: BatchingPlan,
                          phase: str | None = None, kv_policy: str = "offload") -> float:
    """|simulated makespan - critical-path estimate| / estimate under even routing (exec_sim.py:347-360)."""
    wl = wl.with_phase(phase or wl.phase)
    est = build_schedule(spec, hw, latency, wl, plan, kv_policy=kv_policy).critical_path()
    sim = simulate_plan(spec, hw, latency, wl, plan, RoutingModel("even"), kv_policy=kv_policy)
    return abs(sim.makespan - est) / est
